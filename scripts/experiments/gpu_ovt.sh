# per-rank timeline of the overlapped pipeline at 4 GPUs (cfg2, cfg5)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for c in cfg2 cfg5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29951 scripts/ov_timeline.py $c 24 2>/dev/null | grep '^{'
done
