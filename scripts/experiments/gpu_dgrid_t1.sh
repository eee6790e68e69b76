# target-1 dispatch grid beside the TMA-engine return copy: lean 296 (default) / 592 / 1184 CTAs, and 1184 with smem staging (+1184)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do for g in def -592 -1184 1184; do
  if [ $g = def ]; then E=""; else E="MUX_DISPATCH_GRID=$g"; fi
  env $E python bench.py --config target1 --no-nested --no-e2e --no-comparator > gpurun_out/dg.json 2>/dev/null
  echo "grid=$g $(python -c "import json; d=json.loads(open('gpurun_out/dg.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), d['stages'])")"
done; done
