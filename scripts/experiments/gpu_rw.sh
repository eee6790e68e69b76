# balance methods at 2 and 4 GPUs (cfg2 and cfg5): lpt_local (default) vs lpt_local_rw vs lpt
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do for m in lpt_local lpt_local_rw lpt; do for c in cfg2 cfg5; do
  n=4
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29931 bench.py --gpus $n --config $c --method $m --no-nested --no-e2e > gpurun_out/rw.json 2>/dev/null
  echo "$c $m n=$n $(python -c "import json; d=json.loads(open('gpurun_out/rw.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), d['stages'], d['balance']['post_imbalance'])")"
done; done; done
