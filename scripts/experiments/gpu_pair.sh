# full check with the CTA-pair GEMM default: 1-GPU suite, multi suite, benches
N=${1:-4}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest -q -x tests -m gpu -k "not multi" > gpurun_out/p1.log 2>&1; tail -1 gpurun_out/p1.log
timeout 1200 python -m pytest -q -x tests/test_gpu_multi.py > gpurun_out/p2.log 2>&1; tail -1 gpurun_out/p2.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/b_cfg2.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/b_cfg2.json').read()); print('cfg2 n1', round(d['value']/1e6,1), d['ms_per_step'], round(d['roofline']['achieved'],1), round(d['e2e']['value']/1e6,1))"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for n in 2 $N; do $T $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n 2>/dev/null | tail -1 > gpurun_out/b_cfg2_n$n.json; python -c "import json; d=json.loads(open('gpurun_out/b_cfg2_n$n.json').read()); print('cfg2 n$n', round(d['value']/1e6,1), d['ms_per_step'], round(d['roofline']['achieved'],1), round(d['e2e']['value']/1e6,1))"; done
