# return/gradient copies through the TMA engine (MUX_COPY_BULK=1): parity, then target-1 A/B
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_COPY_BULK=1 timeout 900 python -m pytest tests/test_gpu_dataplane.py tests/test_gpu_emulated_world.py -q -x 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
for i in 1 2 3; do for b in 0 1; do
  MUX_COPY_BULK=$b python bench.py --config target1 --no-nested --no-e2e > gpurun_out/cb.json 2>/dev/null
  echo "bulk=$b $(python -c "import json; d=json.loads(open('gpurun_out/cb.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(r['achieved'],1), round(r['frac'],3), d['stages'])")"
done; done
