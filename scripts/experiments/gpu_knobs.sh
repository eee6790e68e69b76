# copy-kernel grab permutation A/B at N GPUs (cfg5 projector off; target1 at N=1)
N=${1:-4}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555"
for perm in 0 1 0 1; do
  MUX_COPY_PERMUTE=$perm MUX_BENCH_CONFIG=cfg5 timeout 600 $T bench.py --gpus $N --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 n$N permute $perm', round(d['value']/1e6,1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages'].items()})"
done
for perm in 0 1; do
  MUX_COPY_PERMUTE=$perm MUX_BENCH_CONFIG=target1 timeout 600 python bench.py --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('target1 permute $perm', round(d['value']/1e6,1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages'].items()})"
done
