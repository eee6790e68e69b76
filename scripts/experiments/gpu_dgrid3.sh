# overlapped dispatch grid beside a return copy: lean 2/SM (-296) vs 3/SM (-444, new default), target-1 x3 and cfg5 at 2 GPUs x2
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do for g in -296 -444; do
  MUX_DISPATCH_GRID=$g python bench.py --config target1 --no-nested --no-e2e --no-comparator > gpurun_out/dg.json 2>/dev/null
  echo "t1 grid=$g $(python -c "import json; d=json.loads(open('gpurun_out/dg.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4))")"
  if [ $i -lt 3 ]; then
  MUX_DISPATCH_GRID=$g timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29992 bench.py --gpus 2 --config cfg5 --no-nested --no-e2e > gpurun_out/dg.json 2>/dev/null
  echo "cfg5 n=2 grid=$g $(python -c "import json; d=json.loads(open('gpurun_out/dg.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4))")"
  fi
done; done
