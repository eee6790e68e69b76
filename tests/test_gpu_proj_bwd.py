"""Projector backward (csrc/proj_bwd.cu, tcgen05) against a torch fp32 reference of
the same products (SPEC.md:411 gradient path):

    dX = G W,  dW = G^T X,  db = sum_m G[m, :]

Tolerance (stated): |gpu - ref_fp32| <= 2^-7 |ref_fp32| + atol, with
atol = 1e-3 for dX (K = 4096-long dot products of unit-scale rows) and
atol = 1e-3 * sqrt(M) for dW / db (M-long sums); the GPU accumulates in fp32
(a different order) and rounds once to bf16."""

import ctypes as C
import math

import pytest
import torch

from paper_2605_08962_b200 import _lib

pytestmark = pytest.mark.gpu
RTOL = 2.0 ** -7


def _check(got, ref, atol, what):
    err = (got.float() - ref).abs()
    tol = RTOL * ref.abs() + atol
    assert bool((err <= tol).all()), f"{what}: max excess {float((err - tol).max())}"


def run_bwd(M, K, N, M_max=None, device_count=False, seed=0, stale=True):
    M_max = M_max or M
    g = torch.Generator(device="cuda").manual_seed(seed)
    G = torch.randn(M_max, N, device="cuda", generator=g).to(torch.bfloat16)
    X = torch.randn(M_max, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    if stale and M_max > M:  # rows past M hold garbage (NaN): they must not leak in
        G[M:] = float("nan")
        X[M:] = float("nan")
    L = _lib.lib()
    ws = torch.empty(L.mux_proj_backward_workspace(K, N, 0), dtype=torch.uint8, device="cuda")
    dx = torch.full((max(M_max, 1), K), 7.0, device="cuda").to(torch.bfloat16)
    dw = torch.empty(N, K, dtype=torch.bfloat16, device="cuda")
    db = torch.empty(N, dtype=torch.bfloat16, device="cuda")
    m_dev = torch.tensor([M], dtype=torch.int64, device="cuda") if device_count else None
    _lib.check(L.mux_proj_backward(G.data_ptr(), X.data_ptr(), W.data_ptr(),
                                   M_max if device_count else M,
                                   m_dev.data_ptr() if device_count else None, K, N,
                                   dx.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(),
                                   ws.numel(), 0, C.c_void_p(torch.cuda.current_stream()
                                                             .cuda_stream)), "bwd")
    torch.cuda.synchronize()
    Gf, Xf, Wf = G[:M].float(), X[:M].float(), W.float()
    _check(dx[:M], Gf @ Wf, 1e-3, "dX")
    if M_max > M:
        assert bool((dx[M:].float() == 7.0).all()), "dX rows past M written"
    at = 1e-3 * math.sqrt(max(M, 1))
    _check(dw, Gf.t() @ Xf, at, "dW")
    _check(db, Gf.sum(0), at, "db")


@pytest.mark.parametrize("M,K,N", [(64, 256, 256), (1000, 256, 512), (4097, 1280, 4096),
                                   (43355, 1280, 4096), (300, 512, 768)])
def test_backward_numerics(cuda_device, M, K, N):
    run_bwd(M, K, N)


def test_backward_device_count_and_stale_rows(cuda_device):
    """The row count read on the device (plan header), stale NaN rows past it:
    the K-block tail is zeroed before the dW reduction and dX rows past M stay."""
    run_bwd(1234, 1280, 4096, M_max=2000, device_count=True)
    run_bwd(0, 256, 256, M_max=128, device_count=True)


def test_backward_rejects_bad_shapes(cuda_device):
    L = _lib.lib()
    assert L.mux_proj_backward(None, None, None, 10, None, 100, 256, None, None, None, None, 0, 0,
                               None) == _lib.MUX_ERR_VALUE


def test_muxpath_projector_backward_after_grad_return(cuda_device):
    """MuxPath: dY at the placeholder rows returned to encoder order
    (grad_return), then projector_backward with the row count from the plan
    header, against torch on the same rows."""
    import numpy as np

    from oracle import planner as oplan
    from paper_2605_08962_b200 import configs, planner
    from paper_2605_08962_b200.dataplane import MuxPath
    from tests.helpers import golden_steps
    from tests.test_gpu_planner import to_table

    for nm, st, t, _ in golden_steps():
        if nm == "cfg2" and st["world"] == 1:
            break
    cap, gbs = configs.CAPACITY, st["gbs"]
    d_in, d_enc, d_llm = configs.D_IN, configs.D_ENC, configs.D_LLM
    path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_enc=d_enc, d_llm=d_llm,
                   projector=True)
    gen = torch.Generator(device="cuda").manual_seed(3)
    W = (torch.randn(d_llm, d_enc[0], device="cuda", generator=gen) / 36).to(torch.bfloat16)
    path.set_projector(0, W, None)
    path.set_projector(1, W, None)
    table = to_table(t)
    dtab = planner.DeviceTable(table, "cuda")
    plan = path.plan(dtab)
    plan.check(table)
    o = oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, "lpt")
    path.encode_standin(plan, dtab)
    n = int(o["llm_rows"][0])
    dy = torch.randn(n, d_llm, device="cuda", generator=gen).to(torch.bfloat16)
    path.grad_return(plan, dy)
    M = int(o["recv_rows"][0, 0])
    Gr = path.grad_view(0, M).clone()
    X = path.enc_view(0, M).clone()
    dx, dw, db = path.projector_backward(0, plan=plan)
    torch.cuda.synchronize()
    # G really is dY at the placeholder rows, in encoder order
    rows = np.concatenate([np.arange(dr, dr + k) for (i, s, r, dr, k) in
                           sorted(o["pieces"], key=lambda p: p[1]) if o["group"][i] == 0])
    assert torch.equal(Gr, dy[torch.from_numpy(rows).cuda()])
    Gf, Xf = Gr.float(), X.float()
    _check(dx[:M], Gf @ W.float(), 1e-3, "dX")
    _check(dw, Gf.t() @ Xf, 1e-3 * math.sqrt(M), "dW")
    _check(db, Gf.sum(0), 1e-3 * math.sqrt(M), "db")
