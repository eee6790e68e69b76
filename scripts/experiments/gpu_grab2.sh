python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for kv in "32768 0" "16384 0" "65536 0" "32768 592" "32768 2368" "16384 2368"; do set -- $kv
  MUX_CHUNK_BYTES=$1 MUX_COPY_GRID=$2 MUX_BENCH_CONFIG=target1 python bench.py --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('target1 chunk $1 grid $2', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['dominant_ms'],4))"
done
