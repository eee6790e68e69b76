# NVLink engine A/B (gpurun --gpus 4): ring / all-to-all / local with SM stores vs TMA bulk
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29800 + n)) scripts/nvlink_probe2.py 256 2>&1 | grep '^{' | tee gpurun_out/nvl2_n$n.json
done
