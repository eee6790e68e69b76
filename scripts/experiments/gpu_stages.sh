# pair-GEMM ring depth A/B (rebuilds between variants)
for st in 6 4 5 6 4 5; do
  MUX_NVCC_DEFS="-DMUX_PAIR_STAGES=$st" python -m paper_2605_08962_b200.build > gpurun_out/build_$st.log 2>&1 || { echo "build $st failed"; continue; }
  python bench.py --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stages $st', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved'],1))"
done
