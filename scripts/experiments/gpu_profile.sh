# single-GPU bench lines + launch lists of the timed region (NVTX range "timed")
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1
python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
MUX_BENCH_CONFIG=target1 python bench.py > gpurun_out/b_t1.json 2> gpurun_out/b_t1.err
python bench.py --impl reference > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
for c in cfg2 target1; do
  MUX_BENCH_SOAK_MS=0 MUX_BENCH_CONFIG=$c python bench.py --steps 4 --warmup 3 --no-e2e > gpurun_out/plain_$c.log 2>&1 && \
  MUX_BENCH_SOAK_MS=0 MUX_BENCH_CONFIG=$c ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --steps 4 --warmup 3 --no-e2e > gpurun_out/ncu_l_$c.log 2>&1
done
echo ok
