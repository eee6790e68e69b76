# pair-GEMM epilogue with TMA tensor stores (build/ab/lib_epitma.so) at one GPU: numerics, then A/B
MUX_LIB_PATH=build/ab/lib_epitma.so timeout 600 python -m pytest tests/test_gpu_proj.py tests/test_gpu_proj_bwd.py -q -x 2>&1 | tail -2
MUX_LIB_PATH=build/ab/lib_epitma.so python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2 3; do for v in default epitma; do
  if [ $v = default ]; then L=""; else L=build/ab/lib_$v.so; fi
  echo "$v: $(MUX_LIB_PATH=$L python scripts/gemm_probe.py 2>&1 | head -1 | cut -c1-100)"
  MUX_LIB_PATH=$L python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/et.json 2>/dev/null
  echo "  step $v: $(python -c "import json; d=json.loads(open('gpurun_out/et.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['roofline']['achieved'],1))")"
done; done
