"""Projector backward at the cfg2 shape (M = 43355 encoder rows, d_enc 1280,
d_llm 4096): per-kernel CUDA-event times of dX (pair GEMM on W^T) and dW (+ db)
and the combined launch, for ncu launch lists and A/B runs."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_08962_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 43355
K, N, reps = 1280, 4096, 10
L = _lib.lib()
g = torch.Generator(device="cuda").manual_seed(0)
G = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
X = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
W = (torch.randn(N, K, device="cuda", generator=g) / 36).to(torch.bfloat16)
ws = torch.empty(L.mux_proj_backward_workspace(K, N, 0), dtype=torch.uint8, device="cuda")
dx = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
dw = torch.empty(N, K, dtype=torch.bfloat16, device="cuda")
db = torch.empty(N, dtype=torch.bfloat16, device="cuda")
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


rows = torch.randperm(M, device="cuda").to(torch.int64)  # gathered variants: G = dY[rows]
gathered = hasattr(L, "mux_proj_backward_rows")


def run(which):
    ptrs = (dx.data_ptr() if "x" in which else None, dw.data_ptr() if "w" in which else None,
            db.data_ptr() if "w" in which and "n" not in which else None)
    if "g" in which:
        _lib.check(L.mux_proj_backward_rows(G.data_ptr(), M, rows.data_ptr(), X.data_ptr(),
                                            W.data_ptr(), M, None, K, N, *ptrs, ws.data_ptr(),
                                            ws.numel(), 0, s))
    else:
        _lib.check(L.mux_proj_backward(G.data_ptr(), X.data_ptr(), W.data_ptr(), M, None, K, N,
                                       *ptrs, ws.data_ptr(), ws.numel(), 0, s))


for which in ("x", "w", "wn", "xw") + (("xg", "wng", "wg", "xwg") if gathered else ()):
    for _ in range(3):
        run(which)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run(which)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    fl = 2.0 * M * K * N * len(which.replace("n", "").replace("g", ""))
    print(f"{which}: {ms:.4f} ms  {fl / ms / 1e9:.1f} TFLOP/s", flush=True)
