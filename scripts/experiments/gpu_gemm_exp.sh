# forward GEMM: ring depth 5/6 and the L2 policy of A, in isolation and in the cfg2 step
for i in 1 2; do for v in default gs5 gs6 ganorm gs6anorm; do
  if [ $v = default ]; then L=""; else L=build/ab/lib_$v.so; fi
  echo "$v: $(MUX_LIB_PATH=$L python scripts/gemm_probe.py 2>&1 | head -1 | cut -c1-90)"
done; done
for i in 1 2; do for v in default gs6 ganorm; do
  if [ $v = default ]; then L=""; else L=build/ab/lib_$v.so; fi
  MUX_LIB_PATH=$L python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/ge.json 2>/dev/null
  echo "step $v: $(python -c "import json; d=json.loads(open('gpurun_out/ge.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['roofline']['achieved'],1))")"
done; done
