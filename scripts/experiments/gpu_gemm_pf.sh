# forward GEMM A/B: L2 prefetch of the next tile's A rows (MUX_GEMM_PREFETCH 0/1), cfg2 at N=1
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do for pf in 0 1; do
  MUX_GEMM_PREFETCH=$pf python bench.py --no-nested --no-e2e > gpurun_out/pf$pf.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pf$pf.json').read().strip().splitlines()[-1]); r=d['roofline']; c=d.get('comparator',{}); print('pf=$pf', round(d['value']/1e6,2), round(r['achieved'],1), round(r['frac'],3), r['peak'], 'cublas', round(c.get('cublas_gemm_only_tflops',0),1), 'bwd', round(d['backward']['tflops'],1))"
done; done
MUX_GEMM_PREFETCH=0 python scripts/bwd_probe.py | head -1; MUX_GEMM_PREFETCH=1 python scripts/bwd_probe.py | head -1
