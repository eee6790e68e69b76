# round-end measurement set (run with gpurun --gpus 4): single-GPU lines, launch
# lists, 2/4-GPU lines, variants
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
bash scripts/gpu_profile.sh > /dev/null 2>&1
for f in b_cfg2 b_t1 b_ref; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,3), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'))"; done
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for cfg in cfg2 cfg5; do for n in 2 4; do
  MUX_BENCH_CONFIG=$cfg timeout 600 $T $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n 2>/dev/null | tail -1 > gpurun_out/b_${cfg}_n$n.json
  python -c "import json; d=json.loads(open('gpurun_out/b_${cfg}_n$n.json').read()); print('$cfg n$n', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1), round(d['e2e']['value']/1e6,1))"
done; done
bash scripts/gpu_variants.sh 4 2>&1 | tail -6
