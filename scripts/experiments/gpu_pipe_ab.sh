# --pipeline 1 vs 2 at one GPU (cfg2 and target-1), alternating; then smoke
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2 3; do for pl in 1 2; do for c in cfg2 target1; do
  python bench.py --config $c --pipeline $pl --no-nested --no-e2e --no-comparator > gpurun_out/pl.json 2>/dev/null
  echo "$c pipeline=$pl $(python -c "import json; d=json.loads(open('gpurun_out/pl.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))")"
done; done; done
