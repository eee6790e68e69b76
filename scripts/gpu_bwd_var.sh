# dW GEMM variants (build/ab/lib_*.so): ring depth 6, 3D TMA boxes; numerics + probe
for v in s6 t3 t3s6; do
  echo "--- $v"; MUX_LIB_PATH=build/ab/lib_$v.so timeout 300 python -m pytest tests/test_gpu_proj_bwd.py -q -x 2>&1 | tail -1
done
for i in 1 2; do for v in default s6 t3 t3s6; do
  if [ $v = default ]; then L=""; else L=build/ab/lib_$v.so; fi
  echo "$v $(MUX_LIB_PATH=$L python scripts/bwd_probe.py 2>&1 | grep -E '^(x|wn):' | tr '\n' ' ')"
done; done
