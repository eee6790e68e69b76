# overlapped dispatch grid (lean CTAs beside the GEMM): 296 (default) vs 148 vs 74, cfg2 at one GPU
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do for g in -296 -148 -74; do
  MUX_DISPATCH_GRID=$g python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/dg.json 2>/dev/null
  echo "grid=$g $(python -c "import json; d=json.loads(open('gpurun_out/dg.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['roofline']['achieved'],1))")"
done; done
