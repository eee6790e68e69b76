# round-2 start: validate the restored tree on one B200 (smoke, -m gpu suite, bench lines)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/s_pytest.log 2>&1; tail -1 gpurun_out/s_pytest.log
python bench.py > gpurun_out/s_cfg2_n1.json 2>gpurun_out/s_cfg2_n1.err
MUX_BENCH_CONFIG=target1 python bench.py > gpurun_out/s_t1_n1.json 2>gpurun_out/s_t1.err
python bench.py --impl reference > gpurun_out/s_ref_n1.json 2>gpurun_out/s_ref.err
tail -c 3000 gpurun_out/s_cfg2_n1.json; tail -c 1500 gpurun_out/s_t1_n1.json; tail -c 800 gpurun_out/s_ref_n1.json
