# projector backward: db on a side stream beside the GEMMs vs in order (previous build)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_proj_bwd.py -q -x 2>&1 | tail -1
for i in 1 2 3; do for v in new head2; do
  if [ $v = new ]; then L=""; else L=build/ab/lib_$v.so; fi
  echo "$v $(MUX_LIB_PATH=$L python scripts/bwd_probe.py 2>&1 | grep -E '^(w|xw):' | tr '\n' ' ')"
done; done
