# guided grab tail (MUX_COPY_TAIL): multi-GPU parity with it on, then cfg5 A/B at 2 and 4 GPUs
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_COPY_TAIL=2 timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x -k "not full" 2>&1 | tail -2
for i in 1 2; do for t in 0 1 2 4; do for n in 2 4; do
  MUX_COPY_TAIL=$t timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2999$n bench.py --gpus $n --config cfg5 --no-nested --no-e2e > gpurun_out/t4.json 2>/dev/null
  echo "tail=$t n=$n $(python -c "import json; d=json.loads(open('gpurun_out/t4.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['nvlink']['return']['gbs'],1), round(d['roofline']['dominant_ms'],4))")"
done; done; done
