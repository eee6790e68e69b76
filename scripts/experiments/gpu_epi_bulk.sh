# pair GEMM epilogue by TMA bulk row copies (build/ab/lib_bulk5.so, ring 5) vs the
# register stores (default ring 6; lib_p5 = ring 5): numerics, then cfg2 at 1 / 2 / 4 GPUs
MUX_LIB_PATH=build/ab/lib_bulk5.so timeout 600 python -m pytest tests/test_gpu_proj.py -q -x 2>&1 | tail -1
MUX_LIB_PATH=build/ab/lib_bulk5.so timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "proj" 2>&1 | tail -1
for i in 1 2; do for v in p6 p5 bulk5; do
  if [ $v = p6 ]; then L=""; else L=build/ab/lib_$v.so; fi
  for n in 1 2 4; do
    if [ $n = 1 ]; then
      MUX_LIB_PATH=$L python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/eb.json 2>/dev/null
    else
      MUX_LIB_PATH=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2991$n bench.py --gpus $n --no-nested --no-e2e > gpurun_out/eb.json 2>/dev/null
    fi
    echo "$v n=$n $(python -c "import json; d=json.loads(open('gpurun_out/eb.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))")"
  done
done; done
