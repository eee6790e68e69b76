python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29941 bench.py --gpus 2 > gpurun_out/n2.json 2>gpurun_out/n2.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/n2.json").read().strip().splitlines()[-1])
for nm, r in (("cfg2", d), ("cfg5", d["cfg5"])):
    nv = r["roofline"]["nvlink"]
    print(nm, round(r["value"]/1e6, 2), round(r["ms_per_step"], 4), "ret gbs", round(nv["return"]["gbs"], 1), round(nv["return"]["frac_of_peak"], 3), nv["return"]["frac_of_alltoall"], nv["probe"])
PY
