# data-path variants at N GPUs: Ulysses vs CpHybrid (cfg4, sp=4), LSSP (cfg5),
# gradient-return stage.  One JSON line each under gpurun_out/var_*.json
N=${1:-4}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544"
run() {  # name config args...
  local nm=$1 cfg=$2; shift 2
  MUX_BENCH_CONFIG=$cfg timeout 600 $T bench.py --gpus $N --no-e2e "$@" > gpurun_out/var_$nm.json 2> gpurun_out/var_$nm.err
  python -c "import json; d=json.loads(open('gpurun_out/var_$nm.json').read().strip().splitlines()[-1]); print('$nm', round(d['value']/1e6,1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages'].items()})"
}
run cfg4_ulysses cfg4
run cfg4_cp cfg4 --reshard cp_hybrid
run cfg5_base cfg5
run cfg5_lssp4096 cfg5 --lssp-eta 4096
run cfg5_lssp4096_g2 cfg5 --lssp-eta 4096 --lssp-sp 2
run cfg2_base cfg2
