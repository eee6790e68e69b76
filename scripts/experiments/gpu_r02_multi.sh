# round 2 (gpurun --gpus 4): whole -m gpu suite (multi-GPU workers at 2-4 ranks, full
# widths included), then the default bench line at 2 and 4 GPUs (nested cfg5 + NVLink roofline)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/m_pytest.log 2>&1; tail -5 gpurun_out/m_pytest.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + n)) bench.py --gpus $n > gpurun_out/m_bench_n$n.json 2> gpurun_out/m_bench_n$n.err
  echo "bench n=$n rc=$?"; tail -3 gpurun_out/m_bench_n$n.err
  python - $n <<'PY'
import json, sys
n = sys.argv[1]
d = json.loads(open(f"gpurun_out/m_bench_n{n}.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("cfg2", n, round(d["value"]/1e6, 2), round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"]/1e6, 2), "frac", round(r["frac"], 3))
c = d.get("cfg5")
if c:
    rr = c["roofline"]; nv = rr["nvlink"]
    print(" cfg5", n, round(c["value"]/1e6, 2), round(c["ms_per_step"], 4), "bound", rr["bound"], "frac", round(rr["frac"], 3))
    print("  return", {k: nv["return"][k] for k in ("remote_bytes_max_rank", "exchange_ms", "gbs", "frac_of_peak", "frac_of_900", "vs_nccl")})
    print("  dispatch", {k: nv["dispatch"][k] for k in ("remote_bytes_max_rank", "exchange_ms", "gbs", "frac_of_peak")})
    print("  probe", nv["probe"], "nccl", nv["nccl_all_to_allv"])
PY
done
