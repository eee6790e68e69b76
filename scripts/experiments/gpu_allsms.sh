# pipelined GEMM on all 148 SMs (planner CTA co-resident) vs 147 SMs: cfg2 at N=1, alternating
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do for a in 0 1; do
  MUX_GEMM_ALL_SMS=$a python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/as$a.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/as$a.json').read().strip().splitlines()[-1]); r=d['roofline']; print('all_sms=$a', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(r['achieved'],1), round(r['frac'],3), d['stages']['plan_ms'])"
done; done
