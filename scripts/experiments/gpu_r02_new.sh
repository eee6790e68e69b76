# round 2: the new single-GPU tests, then the default bench line
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -k "${PYTEST_K:-bwd or streaming or captured or failure or assemble or reorder}" > gpurun_out/n_pytest.log 2>&1; tail -5 gpurun_out/n_pytest.log
grep -E "^E |Error" gpurun_out/n_pytest.log | head -20
timeout 600 python bench.py > gpurun_out/n_bench.json 2>gpurun_out/n_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/n_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/n_bench.json").read().strip().splitlines()[-1])
print("cfg2", round(d["value"]/1e6, 3), d["ms_per_step"], "frac", d["roofline"]["frac"], "bwd", d.get("backward"))
t = d.get("target1")
print("target1", round(t["value"]/1e6, 3), t["ms_per_step"], t["roofline"]["frac"])
PY
