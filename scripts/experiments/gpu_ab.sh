# A/B --pipeline 1 vs 2 at N GPUs (cfg2, cfg5)
N=${1:-2}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29566"
for cfg in cfg2 cfg5; do for rep in 1 2; do for pl in 1 2; do
  MUX_BENCH_CONFIG=$cfg timeout 600 $T bench.py --gpus $N --no-e2e --pipeline $pl 2>gpurun_out/ab_err_$pl.log | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg n$N p$pl', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1), d['clocks']['reasons'])"
done; done; done
