python scripts/cublas_probe.py > gpurun_out/cb_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"gemm|nvjet|sm100|cutlass|xmma" -s 2 -c 1 -o gpurun_out/r02_cublas python scripts/cublas_probe.py > gpurun_out/cb_ncu.log 2>&1
echo rc=$?
