# confirm the grab rule: N=1 target1/cfg2, N=4 cfg5 and cfg2
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for cfg in target1 cfg2; do for rep in 1 2; do
  MUX_BENCH_CONFIG=$cfg python bench.py --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg n1', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['dominant_ms'],4))"
done; done
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29577"
for cfg in cfg5 cfg2; do
  MUX_BENCH_CONFIG=$cfg $T bench.py --gpus 4 --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg n4', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['dominant_ms'],4))"
done
timeout 600 python -m pytest -q -x tests/test_gpu_dataplane.py tests/test_gpu_proj.py 2>&1 | tail -1
