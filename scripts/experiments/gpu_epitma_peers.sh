# TMA-store epilogue into NVLink-peer LLM buffers (gpurun --gpus 4): parity first, then A/B
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -x -k "proj" 2>&1 | tail -2 || exit 1
for i in 1 2; do for pe in 1 0; do for n in 2 4; do
  MUX_EPI_TMA_PEERS=$pe timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2998$n bench.py --gpus $n --no-nested --no-e2e > gpurun_out/tp.json 2>/dev/null
  echo "peers=$pe n=$n $(python -c "import json; d=json.loads(open('gpurun_out/tp.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))")"
done; done; done
