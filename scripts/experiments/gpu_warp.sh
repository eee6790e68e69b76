# copy kernel: block-granular vs warp-granular grabbing (chunk sizes)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_COPY_WARP=1 MUX_CHUNK_BYTES=4096 timeout 300 python -m pytest -q -x tests/test_gpu_dataplane.py 2>&1 | tail -1
for cfg in target1 cfg2; do for kv in "0 32768" "1 4096" "1 8192" "1 16384" "0 32768" "1 8192"; do set -- $kv
  MUX_COPY_WARP=$1 MUX_CHUNK_BYTES=$2 MUX_BENCH_CONFIG=$cfg python bench.py --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg warp $1 chunk $2', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['dominant_ms'],4), round(d['stages']['pack_dispatch_ms'],4))"
done; done
