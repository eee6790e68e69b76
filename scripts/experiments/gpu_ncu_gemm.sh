# ncu --set full of the projector GEMM (pair kernel) in the cfg2 bench; plain run first
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_BENCH_SOAK_MS=0 python bench.py --steps 3 --warmup 3 --no-e2e --distinct 2 > gpurun_out/plain_gemm.log 2>&1 && \
MUX_BENCH_SOAK_MS=0 ncu --set full --clock-control none --import-source on -k regex:proj_scatter_pair -c 1 \
  -o gpurun_out/r01_full_gemm_pair python bench.py --steps 3 --warmup 3 --no-e2e --distinct 2 > gpurun_out/ncu_full_gemm_pair.log 2>&1
echo rc=$?
