# pair-GEMM epilogue staging: 6 stages x 1 buffer (default) vs 5 x 1 (lib_s5) vs 5 x 2 (lib_eb2), cfg2 at 1 and 2 GPUs
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_LIB_PATH=build/ab/lib_eb2.so timeout 600 python -m pytest tests/test_gpu_proj.py -q -x 2>&1 | tail -1
for i in 1 2; do for v in def s5 eb2; do
  if [ $v = def ]; then L=""; else L=build/ab/lib_$v.so; fi
  for n in 1 2; do
    if [ $n = 1 ]; then
      MUX_LIB_PATH=$L python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/eb.json 2>/dev/null
    else
      MUX_LIB_PATH=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n --no-nested --no-e2e --no-comparator > gpurun_out/eb.json 2>/dev/null
    fi
    echo "$v n=$n $(python -c "import json; d=json.loads(open('gpurun_out/eb.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))")"
  done
done; done
