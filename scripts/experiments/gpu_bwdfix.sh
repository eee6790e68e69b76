python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_proj_bwd.py tests/test_gpu_proj.py tests/test_gpu_failure.py -q 2>&1 | grep -E "^E |FAILED|passed|failed" | head
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python scripts/bwd_probe.py | grep -E "^(x|w|xw):"
