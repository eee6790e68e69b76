"""Projector GEMM vs cuBLAS on the same shapes (one GPU): our CTA-pair tcgen05
kernel (mux_proj_scatter, identity row map and with a random row scatter) and
torch.addmm (cuBLAS), bf16 in / fp32 accumulate / bf16 out, CUDA events, 20 reps
after warm-up, inputs N(0,1)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_08962_b200 import _lib  # noqa: E402

L = _lib.lib()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ev_time(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for (M, K, N) in ((43355, 1280, 4096), (52502, 1280, 4096), (8192, 8192, 8192),
                  (43355, 4096, 1280)):
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)
    Y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    base = torch.tensor([Y.data_ptr()], dtype=torch.int64, device="cuda")
    perm = torch.randperm(M, device="cuda")
    fl = 2.0 * M * K * N
    ours = ev_time(lambda: _lib.check(L.mux_proj_scatter(X.data_ptr(), W.data_ptr(), b.data_ptr(),
                                                         M, K, N, None, base.data_ptr(), 0, s)))
    ours_sc = ev_time(lambda: _lib.check(L.mux_proj_scatter(X.data_ptr(), W.data_ptr(),
                                                            b.data_ptr(), M, K, N,
                                                            perm.data_ptr(), base.data_ptr(), 0,
                                                            s)))
    cub = ev_time(lambda: torch.addmm(b, X, W.t(), out=Y))
    print(f"M={M} K={K} N={N}: ours {fl / ours / 1e9:.0f} TFLOP/s ({ours:.4f} ms), ours+scatter "
          f"{fl / ours_sc / 1e9:.0f}, cuBLAS addmm {fl / cub / 1e9:.0f} ({cub:.4f} ms)", flush=True)
