# round 2, one GPU: smoke, whole -m gpu suite, default bench line (nested target-1), reference arm
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/f1_pytest.log 2>&1; tail -3 gpurun_out/f1_pytest.log
grep -E "^(FAILED|ERROR)" gpurun_out/f1_pytest.log | head
timeout 900 python bench.py > gpurun_out/f1_bench.json 2>gpurun_out/f1_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/f1_ref.json 2>gpurun_out/f1_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/f1_bench.json").read().strip().splitlines()[-1])
print("cfg2", round(d["value"]/1e6, 2), round(d["ms_per_step"], 4), "frac", round(d["roofline"]["frac"], 3), "e2e", round(d["e2e"]["value"]/1e6, 2), d["e2e"]["variants"])
print(" comparator", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d["comparator"].items() if k != "note"})
print(" backward", round(d["backward"]["ms"], 4), round(d["backward"]["tflops"], 1))
t = d["target1"]
print("target1", round(t["value"]/1e6, 2), round(t["ms_per_step"], 4), "frac", round(t["roofline"]["frac"], 3), "e2e", round(t["e2e"]["value"]/1e6, 2), t["e2e"]["variants"])
r = json.loads(open("gpurun_out/f1_ref.json").read().strip().splitlines()[-1])
print("ref", round(r["value"]/1e6, 4), r["ms_per_step"], r["cpu_baseline"]["sample"][:160], r["cpu_baseline"].get("cpu_model"), r["config"] == d["config"])
PY
