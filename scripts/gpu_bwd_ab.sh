# projector backward: probe timing + the backward tests
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
python scripts/bwd_probe.py
timeout 600 python -m pytest tests -q -m gpu -k "bwd or assemble" 2>&1 | tail -3
