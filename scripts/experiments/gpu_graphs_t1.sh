# target-1 at one GPU: eager pipelined loop vs one CUDA graph per step (--graphs 1)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do for gr in 0 1; do
  python bench.py --config target1 --graphs $gr --no-nested --no-e2e > gpurun_out/gt.json 2>/dev/null
  echo "graphs=$gr $(python -c "import json; d=json.loads(open('gpurun_out/gt.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), d['impl_config']['launch'])")"
done; done
