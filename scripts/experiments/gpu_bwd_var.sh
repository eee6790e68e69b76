# dW GEMM: L2 prefetch distance (the prefetches double the L2 lookups)
for i in 1 2; do for pf in 8 0 2; do
  echo "prefetch=$pf $(MUX_BWD_PREFETCH=$pf python scripts/bwd_probe.py 2>&1 | grep -E '^(wn|w):' | tr '\n' ' ')"
done; done
