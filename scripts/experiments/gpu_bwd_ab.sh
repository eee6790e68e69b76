# projector backward A/B: the pre-gather build (build/ab/lib_head.so) vs the current one
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do
  echo "--- head"; MUX_LIB_PATH=build/ab/lib_head.so python scripts/bwd_probe.py
  echo "--- new"; python scripts/bwd_probe.py
done
