# pair-GEMM ring 6 (default) vs 5 (build/ab/lib_s5.so), cfg2 at 1 and 4 GPUs, three alternating passes
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do for v in def s5; do
  if [ $v = def ]; then L=""; else L=build/ab/lib_s5.so; fi
  for n in 1 4; do
    if [ $n = 1 ]; then
      MUX_LIB_PATH=$L python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/s5.json 2>/dev/null
    else
      MUX_LIB_PATH=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n --no-nested --no-e2e --no-comparator > gpurun_out/s5.json 2>/dev/null
    fi
    echo "$v n=$n $(python -c "import json; d=json.loads(open('gpurun_out/s5.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))")"
  done
done; done
