# pair-GEMM ring 6 (default now) vs 4 (build/ab/lib_p4.so) at 1, 2 and 4 GPUs, cfg2, alternating
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do for v in p6 p4; do
  if [ $v = p6 ]; then L=""; else L=build/ab/lib_p4.so; fi
  for n in 1 2 4; do
    if [ $n = 1 ]; then
      MUX_LIB_PATH=$L python bench.py --no-nested --no-e2e --no-comparator > gpurun_out/p6.json 2>/dev/null
    else
      MUX_LIB_PATH=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2990$n bench.py --gpus $n --no-nested --no-e2e > gpurun_out/p6.json 2>/dev/null
    fi
    echo "$v n=$n $(python -c "import json; d=json.loads(open('gpurun_out/p6.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))")"
  done
done; done
