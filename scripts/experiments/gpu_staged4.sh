# projector across GPUs at 4 GPUs: fused (GEMM on the encoder rank, epilogue over NVLink) vs staged
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do for m in fused staged; do
  MUX_PROJECTOR_RETURN=$m timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29971 bench.py --gpus 4 --no-nested --no-e2e > gpurun_out/st4.json 2>/dev/null
  echo "$m $(python -c "import json; d=json.loads(open('gpurun_out/st4.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), d['stages'])")"
done; done
