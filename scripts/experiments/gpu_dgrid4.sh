# overlapped dispatch grid at 4 GPUs (cfg2, cfg5): 296 lean CTAs (default) vs 148 vs 74
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do for g in -296 -148 -74; do for c in cfg2 cfg5; do
  MUX_DISPATCH_GRID=$g timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29961 bench.py --gpus 4 --config $c --no-nested --no-e2e > gpurun_out/dg4.json 2>/dev/null
  echo "$c grid=$g $(python -c "import json; d=json.loads(open('gpurun_out/dg4.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4))")"
done; done; done
