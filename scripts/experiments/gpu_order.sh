python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
MUX_GEMM_ORDER=1 timeout 600 python -m pytest -q -x tests/test_gpu_multi.py -k "cfg2 and proj and not staged" 2>&1 | tail -1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for o in 0 1 0 1; do MUX_GEMM_ORDER=$o $T --master-port 2957$o scripts/ov_timeline.py cfg2 24 2>&1 | grep rank | python -c "
import sys,json
rs=[json.loads(l[l.index('{'):]) for l in sys.stdin.read().replace('}{','}\n{').splitlines() if '{' in l]
print('order $o', [round(r['mean_us']['return kernel'],1) for r in sorted(rs,key=lambda r:r['rank'])], rs[0]['mean_us']['period'])"; done
