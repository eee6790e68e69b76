# ncu --set full of target-1's return copy (segcopy, second launch = step 0 return)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_BENCH_SOAK_MS=0 MUX_BENCH_CONFIG=target1 python bench.py --steps 3 --warmup 3 --no-e2e --distinct 2 --pipeline 1 > gpurun_out/plain_t1.log 2>&1 && \
MUX_BENCH_SOAK_MS=0 MUX_BENCH_CONFIG=target1 ncu --set full --clock-control none --import-source on -k regex:segcopy -s 1 -c 1 \
  -o gpurun_out/r01_full_t1_ret python bench.py --steps 3 --warmup 3 --no-e2e --distinct 2 --pipeline 1 > gpurun_out/ncu_full_t1.log 2>&1
echo rc=$?
