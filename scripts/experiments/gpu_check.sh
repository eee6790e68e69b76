# build, single-GPU tests, default bench (cfg2) and target1 bench
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu -k "not multi" > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
MUX_BENCH_CONFIG=target1 python bench.py > gpurun_out/b_t1.json 2> gpurun_out/b_t1.err
echo done
