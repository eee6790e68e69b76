# multi-GPU: parity tests + weak-scaling bench lines (run with gpurun --gpus N)
N=${1:-4}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu -k multi > gpurun_out/pytest_multi.log 2>&1
tail -2 gpurun_out/pytest_multi.log
for cfg in cfg2 cfg5; do
  for n in 2 $N; do
    MUX_BENCH_CONFIG=$cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n \
      > gpurun_out/b_${cfg}_n$n.json 2> gpurun_out/b_${cfg}_n$n.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/b_${cfg}_n$n.json').read().strip().splitlines()[-1]); print('$cfg', $n, d['value']/1e6, d['ms_per_step'], (d.get('e2e') or {}).get('value', 0)/1e6)"
  done
done
