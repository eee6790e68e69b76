python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python -m pytest -q -x tests/test_gpu_proj.py 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for rep in 1 2 3; do python bench.py --no-e2e 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 n1', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))"; done
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29599"
$T bench.py --gpus 4 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 n4', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))"
timeout 600 python -m pytest -q -x tests/test_gpu_multi.py -k "proj" 2>&1 | tail -1
