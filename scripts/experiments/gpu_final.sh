# final validation: smoke, the whole -m gpu suite, bench lines at 1/2/4 GPUs
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_final.log 2>&1; tail -1 gpurun_out/pytest_final.log
python bench.py > gpurun_out/f_cfg2_n1.json 2>/dev/null
MUX_BENCH_CONFIG=target1 python bench.py > gpurun_out/f_t1_n1.json 2>/dev/null
python bench.py --impl reference > gpurun_out/f_ref_n1.json 2>/dev/null
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for n in 2 4; do $T $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n 2>/dev/null | tail -1 > gpurun_out/f_cfg2_n$n.json; done
for f in f_cfg2_n1 f_t1_n1 f_ref_n1 f_cfg2_n2 f_cfg2_n4; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,3), d.get('ms_per_step'), round((d.get('e2e') or {}).get('value',0)/1e6,2), (d.get('roofline') or {}).get('frac'))"; done
