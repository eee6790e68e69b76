# round 2 profiles (one GPU): launch lists of the timed region (cfg2, target-1),
# ncu --set full of the pair GEMM (cfg2), the return copy (target-1) and the dW GEMM.
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for c in cfg2 target1; do
  MUX_BENCH_SOAK_MS=0 python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-nested --no-comparator > gpurun_out/p_plain_$c.log 2>&1 && \
  MUX_BENCH_SOAK_MS=0 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02_launches_$c.csv python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-nested --no-comparator > gpurun_out/p_ncu_l_$c.log 2>&1
  echo "launches $c rc=$?"
done
MUX_BENCH_SOAK_MS=0 python bench.py --steps 3 --warmup 3 --no-e2e --no-nested --no-comparator --distinct 2 > gpurun_out/p_plain_gemm.log 2>&1 && \
MUX_BENCH_SOAK_MS=0 ncu --set full --clock-control none --import-source on -k regex:proj_scatter_pair -c 1 \
  -o gpurun_out/r02_full_gemm_pair python bench.py --steps 3 --warmup 3 --no-e2e --no-nested --no-comparator --distinct 2 > gpurun_out/p_ncu_gemm.log 2>&1
echo "gemm rc=$?"
MUX_BENCH_SOAK_MS=0 python bench.py --config target1 --steps 3 --warmup 3 --no-e2e --no-nested --distinct 2 --pipeline 1 > gpurun_out/p_plain_t1.log 2>&1 && \
MUX_BENCH_SOAK_MS=0 ncu --set full --clock-control none --import-source on -k regex:segcopy -s 1 -c 1 \
  -o gpurun_out/r02_full_t1_ret python bench.py --config target1 --steps 3 --warmup 3 --no-e2e --no-nested --distinct 2 --pipeline 1 > gpurun_out/p_ncu_t1.log 2>&1
echo "t1 rc=$?"
python scripts/bwd_probe.py > gpurun_out/p_plain_bwd.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dw_pair -s 1 -c 1 -o gpurun_out/r02_full_dw python scripts/bwd_probe.py > gpurun_out/p_ncu_dw.log 2>&1
echo "dw rc=$?"
