# split local/remote copy queues: parity, then A/B at 4 GPUs
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest -q -x tests/test_gpu_multi.py -k "cfg5 or cfg3 or cfg4" > gpurun_out/split_test.log 2>&1; tail -1 gpurun_out/split_test.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29599"
for kv in "0 0" "1 296" "1 148" "1 592" "0 0" "1 296"; do set -- $kv
  MUX_COPY_SPLIT=$1 MUX_COPY_REMOTE_CTAS=$2 MUX_BENCH_CONFIG=cfg5 timeout 600 $T bench.py --gpus 4 --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 n4 split $1 rctas $2', round(d['value']/1e6,1), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages'].items()})"
done
