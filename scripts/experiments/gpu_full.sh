# round-end style check on one GPU: build, smoke, full -m gpu suite, default bench
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
python -c "import json; d=json.loads(open('gpurun_out/b_cfg2.json').read()); print('cfg2', round(d['value']/1e6,1), d['ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']/1e6,1))"
MUX_BENCH_CONFIG=target1 python bench.py > gpurun_out/b_t1.json 2> gpurun_out/b_t1.err
python -c "import json; d=json.loads(open('gpurun_out/b_t1.json').read()); print('target1', round(d['value']/1e6,1), d['ms_per_step'], round(d['roofline']['frac'],3), round(d['e2e']['value']/1e6,1))"
python bench.py --impl reference > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; tail -c 300 gpurun_out/b_ref.json
