# mixed local + NVLink copy probe (gpurun --gpus 4)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for args in "170 14" "170 22"; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29811 scripts/nvlink_probe3.py $args 2>&1 | grep -E '^\{|Error'
done
