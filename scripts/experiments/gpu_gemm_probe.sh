python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python scripts/gemm_probe.py
python bench.py --no-nested --no-e2e > gpurun_out/g_bench.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g_bench.json').read().strip().splitlines()[-1]); print(d['value']/1e6, d['roofline']['achieved'], d['comparator'])"
