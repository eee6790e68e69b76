# e2e upload timeline: per-step upload start/end and step-end events (MUX_E2E_TRACE, GPU ms / host enqueue ms)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
python scripts/probes/pinned_upload_probe.py
for st in 16; do
  MUX_E2E_TRACE=1 python bench.py --config cfg2 --steps $st --warmup 3 --no-nested --no-comparator > gpurun_out/e2e_$st.json 2> gpurun_out/e2e_$st.err
  grep "e2e trace" gpurun_out/e2e_$st.err | head -1
  python -c "import json;d=json.loads(open('gpurun_out/e2e_$st.json').read().strip().splitlines()[-1]);print('$st', d['e2e']['variants'], d['e2e']['h2d_bytes_per_step'])"
done
