# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck
TOOL=${TOOL:-memcheck}
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
python scripts/sanitize_smoke.py > gpurun_out/san_plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/san_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python scripts/sanitize_smoke.py > gpurun_out/san_$TOOL.log 2>&1
echo "rc=$?"; tail -8 gpurun_out/san_$TOOL.log
