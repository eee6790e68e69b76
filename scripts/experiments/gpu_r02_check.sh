# round 2: single-GPU tests + default bench line (with nested target1 + comparator) + reference arm
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/c_pytest.log 2>&1; tail -3 gpurun_out/c_pytest.log
python bench.py > gpurun_out/c_bench.json 2>gpurun_out/c_bench.err; echo "bench rc=$?"
tail -5 gpurun_out/c_bench.err
${SKIP_REF:+true} python bench.py --impl reference > gpurun_out/c_ref.json 2>gpurun_out/c_ref.err
python - <<'PY'
import json
for f in ("c_bench", "c_ref"):
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no line", e); continue
    r = d.get("roofline") or {}
    print(f, round(d["value"]/1e6, 3), d.get("ms_per_step"), "e2e", round((d.get("e2e") or {}).get("value", 0)/1e6, 2), "frac", r.get("frac"), r.get("peak"), d.get("comparator"))
    t = d.get("target1")
    if t:
        print("  target1", round(t["value"]/1e6, 3), t["ms_per_step"], "e2e", round(t["e2e"]["value"]/1e6, 2), "frac", t["roofline"]["frac"], t["roofline"].get("frac_of_nominal_8000"))
    print("  config", d.get("config"))
PY
