# projector backward: plain timing, then an ncu launch list and a full capture of dw_pair_kernel
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
python scripts/bwd_probe.py > gpurun_out/bwd_plain.log 2>&1 && cat gpurun_out/bwd_plain.log &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_launches.csv python scripts/bwd_probe.py > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/bwd_launches.csv 2>/dev/null | head -30
ncu --set full --clock-control none --import-source on -k regex:dw_pair -s 2 -c 1 -o gpurun_out/bwd_dw python scripts/bwd_probe.py > gpurun_out/bwd_ncu.log 2>&1; tail -3 gpurun_out/bwd_ncu.log
