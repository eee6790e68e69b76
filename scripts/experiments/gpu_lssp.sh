# LSSP and gradient-return measurements at N GPUs
N=${1:-4}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533"
for eta in -1 4096 1024; do
  MUX_BENCH_CONFIG=cfg5 $T bench.py --gpus $N --no-e2e --lssp-eta $eta > gpurun_out/b_lssp_$eta.json 2> gpurun_out/b_lssp_$eta.err
  python -c "import json; d=json.loads(open('gpurun_out/b_lssp_$eta.json').read().strip().splitlines()[-1]); print('cfg5 n$N eta $eta', round(d['value']/1e6,1), d['ms_per_step'], d['stages'])"
done
MUX_BENCH_CONFIG=cfg2 $T bench.py --gpus $N --no-e2e --lssp-eta 4096 > gpurun_out/b_lssp_cfg2.json 2> gpurun_out/b_lssp_cfg2.err
python -c "import json; d=json.loads(open('gpurun_out/b_lssp_cfg2.json').read().strip().splitlines()[-1]); print('cfg2 n$N eta 4096', round(d['value']/1e6,1), d['ms_per_step'], d['stages'])"
