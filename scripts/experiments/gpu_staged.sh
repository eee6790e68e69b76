# fused vs staged projector return at N GPUs (pair GEMM), pipeline 2 and 1
N=${1:-4}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29588"
for mode in fused staged; do for pl in 2 1; do
  MUX_PROJECTOR_RETURN=$mode timeout 600 $T bench.py --gpus $N --no-e2e --pipeline $pl 2>gpurun_out/st_$mode$pl.err | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 n$N $mode p$pl', round(d['value']/1e6,1), round(d['ms_per_step'],4), d['exchange'])" || tail -3 gpurun_out/st_$mode$pl.err
done; done
