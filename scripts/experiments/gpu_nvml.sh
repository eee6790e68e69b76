# NVML NVLink counters in the bench at 2 GPUs (cfg2 with nested cfg5)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29941 bench.py --gpus 2 --no-e2e > gpurun_out/nvml.json 2>gpurun_out/nvml.err; echo rc=$?
tail -3 gpurun_out/nvml.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/nvml.json").read().strip().splitlines()[-1])
for nm, r in (("cfg2", d), ("cfg5", d["cfg5"])):
    nv = r["roofline"]["nvlink"]
    print(nm, round(r["value"]/1e6, 2), nv.get("nvml_counters"), round(nv["return"]["gbs"], 1))
PY
