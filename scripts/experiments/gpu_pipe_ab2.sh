# default pipeline (auto: 1 for cfg2 at N=1) vs --pipeline 2, alternating, cfg2 at one GPU
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3 4; do for pl in -1 2; do
  python bench.py --pipeline $pl --no-nested --no-e2e --no-comparator > gpurun_out/pl.json 2>/dev/null
  echo "pipeline=$pl $(python -c "import json; d=json.loads(open('gpurun_out/pl.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['impl_config']['planner'])")"
done; done
