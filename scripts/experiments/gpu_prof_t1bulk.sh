# target-1 with the TMA-engine return copy: launch list of the timed region + ncu --set full of one return copy
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
c=target1
MUX_BENCH_SOAK_MS=0 python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-nested --no-comparator > gpurun_out/p_plain_$c.log 2>&1 && \
MUX_BENCH_SOAK_MS=0 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_$c.csv python bench.py --config $c --steps 4 --warmup 3 --no-e2e --no-nested --no-comparator > gpurun_out/p_ncu_l_$c.log 2>&1
echo "launches rc=$?"
MUX_BENCH_SOAK_MS=0 python bench.py --config target1 --steps 3 --warmup 3 --no-e2e --no-nested --distinct 2 --pipeline 1 > gpurun_out/p_plain_t1.log 2>&1 && \
MUX_BENCH_SOAK_MS=0 ncu --set full --clock-control none --import-source on -k regex:segcopy_bulk -s 1 -c 1 \
  -o gpurun_out/r02_full_t1_ret python bench.py --config target1 --steps 3 --warmup 3 --no-e2e --no-nested --distinct 2 --pipeline 1 > gpurun_out/p_ncu_t1.log 2>&1
echo "t1 rc=$?"
