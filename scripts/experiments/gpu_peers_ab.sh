# (a) db on a side stream (one GPU); (b) TMA peer stores on/off at 2 GPUs, alternating, + timelines
bash scripts/experiments/gpu_dbside.sh
for i in 1 2 3; do for pe in 1 0; do
  MUX_EPI_TMA_PEERS=$pe timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29991 bench.py --gpus 2 --no-nested --no-e2e > gpurun_out/pa.json 2>/dev/null
  echo "peers=$pe n=2 $(python -c "import json; d=json.loads(open('gpurun_out/pa.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1), d['stages'])")"
done; done
for pe in 1 0; do
  echo "timeline peers=$pe"
  MUX_EPI_TMA_PEERS=$pe timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29992 scripts/ov_timeline.py cfg2 24 2>/dev/null | grep '^{'
done
