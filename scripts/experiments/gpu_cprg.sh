python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -q -m gpu -k "reorder_groups_and_flops" 2>&1 | tail -3
