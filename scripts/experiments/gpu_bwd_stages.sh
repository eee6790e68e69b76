# dW pair-GEMM ring depth: 4 (default) vs 5 (lib_b5) vs 6 (lib_b6), bwd_probe + bench backward, two alternating passes
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_LIB_PATH=build/ab/lib_b6.so timeout 600 python -m pytest tests/test_gpu_proj_bwd.py -q -x 2>&1 | tail -1
for i in 1 2; do for v in def b5 b6; do
  if [ $v = def ]; then L=""; else L=build/ab/lib_$v.so; fi
  echo "$v: $(MUX_LIB_PATH=$L python scripts/bwd_probe.py 2>/dev/null | tr '\n' ' ')"
  MUX_LIB_PATH=$L python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/bs.json 2>/dev/null
  echo "$v bench: $(python -c "import json; d=json.loads(open('gpurun_out/bs.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['backward']['ms'],4), round(d['backward']['tflops'],1))")"
done; done
