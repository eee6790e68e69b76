# bench lines for every multi-GPU config at 2 and 4 GPUs (cfg3, cfg4) + target1/cfg5 at 1
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for cfg in cfg3 cfg4; do for n in 2 4; do
  MUX_BENCH_CONFIG=$cfg timeout 600 $T $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n 2>/dev/null | tail -1 > gpurun_out/b_${cfg}_n$n.json
  python -c "import json; d=json.loads(open('gpurun_out/b_${cfg}_n$n.json').read()); print('$cfg n$n', round(d['value']/1e6,1), round(d['ms_per_step'],4), d['config']['parallelism'], round(d['e2e']['value']/1e6,1))"
done; done
for cfg in cfg5 cfg3; do
  MUX_BENCH_CONFIG=$cfg python bench.py 2>/dev/null | tail -1 > gpurun_out/b_${cfg}_n1.json
  python -c "import json; d=json.loads(open('gpurun_out/b_${cfg}_n1.json').read()); print('$cfg n1', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['e2e']['value']/1e6,1))"
done
