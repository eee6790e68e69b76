# bench.py option coverage after the round-2 refactor (gpurun --gpus 2)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
run1() { timeout 600 python bench.py --no-nested "$@" > gpurun_out/fl.json 2>gpurun_out/fl.err; echo "n=1 $* rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/fl.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), d['ms_per_step'])" 2>&1 | tail -1)"; }
run2() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29901 bench.py --gpus 2 --no-nested "$@" > gpurun_out/fl.json 2>gpurun_out/fl.err; echo "n=2 $* rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/fl.json').read().strip().splitlines()[-1]); print(round(d['value']/1e6,2), d['ms_per_step'])" 2>&1 | tail -1)"; }
run1 --config target1 --text-embed --no-e2e
run1 --graphs 1 --no-e2e
run1 --pipeline 1 --no-e2e --method kk
run1 --config cfg3 --no-e2e
run2 --config cfg4 --reshard cp_hybrid --no-e2e
run2 --config cfg5 --lssp-eta 4096 --no-e2e
run2 --graphs 1 --no-e2e
run2 --config cfg3 --method lpt_local_rw
