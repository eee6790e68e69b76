# round 2 (gpurun --gpus 4): multi-GPU parity (incl. metadata all-gather, reorder groups,
# full widths), then the default bench line at 2 and 4 GPUs
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 1800 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/m2_pytest.log 2>&1; tail -3 gpurun_out/m2_pytest.log
grep -E "^(FAILED|ERROR)" gpurun_out/m2_pytest.log | head
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700 + n)) bench.py --gpus $n > gpurun_out/m2_bench_n$n.json 2> gpurun_out/m2_bench_n$n.err
  echo "bench n=$n rc=$?"
  python - $n <<'PY'
import json, sys
n = sys.argv[1]
d = json.loads(open(f"gpurun_out/m2_bench_n{n}.json").read().strip().splitlines()[-1])
print("cfg2", n, round(d["value"]/1e6, 2), round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"]/1e6, 2), "frac", round(d["roofline"]["frac"], 3), "bwd", round(d["backward"]["tflops"], 1), d["balance"]["pre_imbalance"], d["balance"]["post_imbalance"])
c = d["cfg5"]; nv = c["roofline"]["nvlink"]
print(" cfg5", n, round(c["value"]/1e6, 2), round(c["ms_per_step"], 4), "nvlink", round(nv["return"]["gbs"], 1), round(nv["return"]["frac_of_peak"], 3), round(nv["return"]["frac_of_900"], 3), "vs_nccl", round(nv["return"]["vs_nccl"], 2), c["balance"]["post_imbalance"], "combined", round(c["roofline"].get("frac_combined_hbm_nvlink") or 0, 3), "e2e", round(c["e2e"]["value"]/1e6, 2) if c.get("e2e") else None)
PY
done
