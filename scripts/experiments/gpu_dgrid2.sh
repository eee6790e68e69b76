# overlapped dispatch grid default (lean 8/SM beside a return copy, 2/SM beside the GEMM): parity + A/B at 1 and 2 GPUs
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "overlap" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_dataplane.py tests/test_gpu_proj.py tests/test_gpu_failure.py -q -x 2>&1 | tail -1
for i in 1 2; do for g in def -296; do
  if [ $g = def ]; then E=""; else E="MUX_DISPATCH_GRID=$g"; fi
  env $E python bench.py --config target1 --no-nested --no-e2e --no-comparator > gpurun_out/dg.json 2>/dev/null
  echo "t1 grid=$g $(python -c "import json; d=json.loads(open('gpurun_out/dg.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4))")"
  env $E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29992 bench.py --gpus 2 --config cfg5 --no-nested --no-e2e > gpurun_out/dg.json 2>/dev/null
  echo "cfg5 n=2 grid=$g $(python -c "import json; d=json.loads(open('gpurun_out/dg.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4))")"
done; done
