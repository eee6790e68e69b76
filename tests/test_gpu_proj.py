"""Projector GEMM (tcgen05) fused with the scatter: numerics against a torch fp32
reference of the same op, and the full cfg2 step against the oracle.

Tolerance (stated): |gpu - ref_fp32| <= 2^-7 * |ref_fp32| + 1e-3, where ref_fp32
is X.float() @ W.float().T + b with fp32 accumulation; the GPU rounds the fp32
accumulator to bf16 once (<= 2^-8 relative) and sums K in a different order."""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2605_08962_b200 import _lib

pytestmark = pytest.mark.gpu
RTOL, ATOL = 2.0 ** -7, 1e-3


def run_proj(M, K, N, R, bias=True, seed=0, world_rows=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    X = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16) if bias else None
    perm = torch.randperm(R, generator=torch.Generator().manual_seed(seed))[:M]
    out = torch.zeros(R, N, dtype=torch.bfloat16, device="cuda")
    row_dst = perm.to(torch.int64).cuda()  # rank 0
    bases = torch.tensor([out.data_ptr()], dtype=torch.int64, device="cuda")
    st = _lib.lib().mux_proj_scatter(X.data_ptr(), W.data_ptr(), b.data_ptr() if bias else None,
                                     M, K, N, row_dst.data_ptr(), bases.data_ptr(), 0,
                                     torch.cuda.current_stream().cuda_stream)
    _lib.check(st)
    torch.cuda.synchronize()
    ref = X.float() @ W.float().t()
    if bias:
        ref = ref + b.float()
    got = out[perm.cuda()].float()
    err = (got - ref).abs()
    tol = RTOL * ref.abs() + ATOL
    assert bool((err <= tol).all()), f"max excess {float((err - tol).max())}"
    untouched = torch.ones(R, dtype=torch.bool)
    untouched[perm] = False
    assert bool((out[untouched.cuda()] == 0).all()), "scatter wrote outside row_dst"
    return float(err.max())


@pytest.mark.parametrize("M,K,N", [(128, 64, 256), (1000, 1280, 512), (4097, 1280, 4096),
                                   (300, 512, 768)])
def test_proj_scatter_numerics(cuda_device, M, K, N):
    run_proj(M, K, N, R=M + 777, bias=(M % 2 == 0))


def test_proj_scatter_device_count(cuda_device):
    """M read from device memory: rows >= *M_dev are neither computed nor stored."""
    M_max, K, N = 1024, 256, 256
    X = torch.randn(M_max, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(M_max, N, dtype=torch.bfloat16, device="cuda")
    row_dst = torch.arange(M_max, dtype=torch.int64, device="cuda")
    bases = torch.tensor([out.data_ptr()], dtype=torch.int64, device="cuda")
    m_dev = torch.tensor([517], dtype=torch.int64, device="cuda")
    st = _lib.lib().mux_proj_scatter_dev(X.data_ptr(), W.data_ptr(), None, M_max, m_dev.data_ptr(),
                                         K, N, row_dst.data_ptr(), bases.data_ptr(), 0,
                                         torch.cuda.current_stream().cuda_stream)
    _lib.check(st)
    torch.cuda.synchronize()
    ref = (X[:517].float() @ W.float().t())
    assert bool(((out[:517].float() - ref).abs() <= RTOL * ref.abs() + ATOL).all())
    assert bool((out[517:] == 0).all())


def test_proj_grouped_two_encoders(cuda_device):
    """Both encoder groups in one launch: different K, device row counts, rows
    of both groups interleaved in one output; an empty group is skipped."""
    g = torch.Generator(device="cuda").manual_seed(9)
    N, R = 512, 3000
    Ks, Mmax, Mdev = (1280, 512), (900, 600), (700, 333)
    Xs = [torch.randn(Mmax[k], Ks[k], device="cuda", generator=g).to(torch.bfloat16)
          for k in range(2)]
    Ws = [(torch.randn(N, Ks[k], device="cuda", generator=g) / Ks[k] ** 0.5).to(torch.bfloat16)
          for k in range(2)]
    b1 = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)
    perm = torch.randperm(R, generator=torch.Generator().manual_seed(2))
    rd = [perm[:Mmax[0]].to(torch.int64).cuda(), perm[1000:1000 + Mmax[1]].to(torch.int64).cuda()]
    mdev = torch.tensor(Mdev, dtype=torch.int64, device="cuda")
    out = torch.zeros(R, N, dtype=torch.bfloat16, device="cuda")
    bases = torch.tensor([out.data_ptr()], dtype=torch.int64, device="cuda")
    groups = (_lib.ProjGroup * 2)(
        _lib.ProjGroup(Xs[0].data_ptr(), Ws[0].data_ptr(), None, Mmax[0], mdev.data_ptr(),
                       Ks[0], 0, rd[0].data_ptr()),
        _lib.ProjGroup(Xs[1].data_ptr(), Ws[1].data_ptr(), b1.data_ptr(), Mmax[1],
                       mdev.data_ptr() + 8, Ks[1], 0, rd[1].data_ptr()))
    _lib.check(_lib.lib().mux_proj_scatter_grouped(groups, 2, N, bases.data_ptr(), 0,
                                                   torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    written = torch.zeros(R, dtype=torch.bool, device="cuda")
    for k in range(2):
        m = Mdev[k]
        ref = Xs[k][:m].float() @ Ws[k].float().t() + (b1.float() if k else 0.0)
        got = out[rd[k][:m]].float()
        assert bool(((got - ref).abs() <= RTOL * ref.abs() + ATOL).all()), f"group {k}"
        written[rd[k][:m]] = True
    assert bool((out[~written] == 0).all()), "rows past *M_dev were stored"
    # an empty group (device count 0) and a dropped one (M_max 0) launch nothing wrong
    out.zero_()
    mdev[0] = 0
    groups[1].M_max = 0
    _lib.check(_lib.lib().mux_proj_scatter_grouped(groups, 2, N, bases.data_ptr(), 0,
                                                   torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert bool((out == 0).all())


def test_proj_rejects_bad_shapes(cuda_device):
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().mux_proj_scatter(None, None, None, 10, 100, 256, None, None, 0, None))


@pytest.mark.parametrize("name,step", [("cfg2", 1), ("target1", 1)])
def test_step_with_projector_matches_oracle(cuda_device, name, step):
    """Full step at ViT-600M -> 7B shapes: plan, pack, stand-in, projector+scatter
    (target1 step 1 has vision and audio rows: both groups in one GEMM launch)."""
    from oracle import dataplane as odp
    from oracle import planner as oplan
    from paper_2605_08962_b200 import configs, planner
    from paper_2605_08962_b200.dataplane import MuxPath
    from tests.helpers import golden_steps
    from tests.test_gpu_planner import to_table

    for nm, st, t, _ in golden_steps():
        if nm != name or st["step"] != step or st["world"] != 1:
            continue
        cap, gbs = configs.CAPACITY, st["gbs"]
        d_in, d_enc, d_llm = configs.D_IN, configs.D_ENC, configs.D_LLM
        o = oplan.plan_step(t, cap, gbs, 1, 1, 1)
        path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_enc=d_enc, d_llm=d_llm,
                       projector=True)
        assert name != "target1" or int(o["recv_rows"][0, 1]) > 0
        g = torch.Generator().manual_seed(3)
        Ws = [(torch.randn(d_llm, d_enc[k], generator=g) / d_enc[k] ** 0.5).to(torch.bfloat16)
              for k in range(2)]
        bs = [torch.randn(d_llm, generator=g).to(torch.bfloat16) for k in range(2)]
        for k in range(2):
            path.set_projector(k, Ws[k].cuda(), bs[k].cuda())
        arenas = [torch.randn(max(int(o["arena_rows"][0, k]), 1), d_in[k], generator=g)
                  .to(torch.bfloat16) for k in range(2)]
        table = to_table(t)
        dtab = planner.DeviceTable(table, "cuda")
        plan = path.plan(dtab)
        plan.check(table)
        path.llm_view().zero_()
        path.dispatch(plan, [a.cuda() for a in arenas])
        path.encode_standin(plan, dtab)
        path.return_scatter(plan)
        torch.cuda.synchronize()
        # reference in torch fp32 on the GPU from the (bit-exact) encoder rows
        n = int(o["llm_rows"][0])
        got = path.llm_view(n).float()
        ref = torch.zeros(n, d_llm, device="cuda")
        for (i, src, dst_rank, dst_row, rows) in o["pieces"]:
            k = int(o["group"][i])
            x = torch.from_numpy(odp.standin(int(t["ids"][i]), int(t["lens"][i]), d_enc[k])
                                 .view(np.int16)).view(torch.bfloat16).cuda()[:rows]
            ref[dst_row:dst_row + rows] = x.float() @ Ws[k].cuda().float().t() + bs[k].cuda().float()
        err = (got - ref).abs()
        assert bool((err <= RTOL * ref.abs() + ATOL).all()), float((err - RTOL * ref.abs()).max())
        mask = torch.zeros(n, dtype=torch.bool, device="cuda")
        for (i, src, dst_rank, dst_row, rows) in o["pieces"]:
            mask[dst_row:dst_row + rows] = True
        assert bool((got[~mask] == 0).all())
        return
    raise AssertionError(f"{name} golden step {step} missing")


@pytest.mark.parametrize("overlap", [False, True])
def test_pipelined_ring_matches_oracle(cuda_device, overlap):
    """The bench's pipelined form (MuxPath.run_pipeline): step k+1 planned on the
    side stream (plan ring, row map built there) while step k moves, and with
    overlap_dispatch its dispatch on the copy stream under step k's projector;
    every step's LLM rows checked."""
    from oracle import planner as oplan
    from paper_2605_08962_b200 import configs, planner
    from paper_2605_08962_b200.dataplane import MuxPath
    from tests.helpers import golden_steps
    from tests.test_gpu_planner import to_table

    steps = [(st, t) for nm, st, t, _ in golden_steps() if nm == "target1" and st["world"] == 1]
    steps = (steps * 3)[:6]  # more steps than ring slots
    cap, gbs = configs.CAPACITY, steps[0][0]["gbs"]
    d_in, d_enc, d_llm = configs.D_IN, configs.D_ENC, 512
    path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_enc=d_enc, d_llm=d_llm,
                   projector=True, method="lpt_local", overlap_dispatch=overlap)
    g = torch.Generator().manual_seed(5)
    Ws = [(torch.randn(d_llm, d_enc[k], generator=g) / d_enc[k] ** 0.5).to(torch.bfloat16).cuda()
          for k in range(2)]
    for k in range(2):
        path.set_projector(k, Ws[k], None)
    tabs = [planner.DeviceTable(to_table(t), "cuda") for _, t in steps]
    os_ = [oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, "lpt_local") for _, t in steps]
    arenas = [[torch.zeros(max(int(o["arena_rows"][0, k]), 1), d_in[k], dtype=torch.bfloat16,
                           device="cuda") for k in range(2)] for o in os_]
    outs = []

    def encoder(k, p, s):
        path.llm_view().zero_()
        path.encode_standin(p, tabs[k], s)

    def after(k, p, s):
        outs.append(path.llm_view(int(os_[k]["llm_rows"][0])).float().clone())

    path.run_pipeline(list(zip(tabs, arenas)), encoder=encoder, after_step=after)
    torch.cuda.synchronize()
    from oracle import dataplane as odp
    for k, ((st, t), o) in enumerate(zip(steps, os_)):
        n = int(o["llm_rows"][0])
        ref = torch.zeros(n, d_llm, device="cuda")
        for (i, src, dst_rank, dst_row, rows) in o["pieces"]:
            q = int(o["group"][i])
            x = torch.from_numpy(odp.standin(int(t["ids"][i]), int(t["lens"][i]), d_enc[q])
                                 .view(np.int16)).view(torch.bfloat16).cuda()
            off = src - int(o["enc_off"][i])
            ref[dst_row:dst_row + rows] = x[off:off + rows].float() @ Ws[q].float().t()
        err = (outs[k] - ref).abs()
        assert bool((err <= RTOL * ref.abs() + ATOL).all()), f"step {k}"


def test_captured_step_graphs_match_oracle(cuda_device):
    """MuxPath.capture_steps (bench --graphs 1): one CUDA graph per distinct step
    (plan of step i+1 on the side stream beside step i's dispatch + projector);
    replayed steps give the projected rows of the fp32 reference."""
    from oracle import dataplane as odp
    from oracle import planner as oplan
    from paper_2605_08962_b200 import configs, planner
    from paper_2605_08962_b200.dataplane import MuxPath
    from tests.helpers import golden_steps
    from tests.test_gpu_planner import to_table

    steps = [(st, t) for nm, st, t, _ in golden_steps() if nm == "target1" and st["world"] == 1]
    steps = steps[:2]
    cap, gbs = configs.CAPACITY, steps[0][0]["gbs"]
    d_in, d_enc, d_llm = configs.D_IN, configs.D_ENC, 512
    path = MuxPath(capacity=cap, gbs=gbs, dp=1, d_in=d_in, d_enc=d_enc, d_llm=d_llm,
                   projector=True, method="lpt")
    g = torch.Generator().manual_seed(8)
    Ws = [(torch.randn(d_llm, d_enc[k], generator=g) / d_enc[k] ** 0.5).to(torch.bfloat16).cuda()
          for k in range(2)]
    for k in range(2):
        path.set_projector(k, Ws[k], None)
    tabs = [planner.DeviceTable(to_table(t), "cuda") for _, t in steps]
    os_ = [oplan.plan_step(t, cap, gbs, 1, 1, 1, 1, "lpt") for _, t in steps]
    arenas = [[torch.zeros(max(int(o["arena_rows"][0, k]), 1), d_in[k], dtype=torch.bfloat16,
                           device="cuda") for k in range(2)] for o in os_]
    graphs = path.capture_steps(tabs, arenas)
    graphs.prime(0)
    for i, ((st, t), o) in enumerate(zip(steps, os_)):
        path.zero_llm()
        path.encode_standin(graphs.plans[i], tabs[i])
        graphs.replay(i)
        torch.cuda.synchronize()
        n = int(o["llm_rows"][0])
        got = path.llm_view(n).float()
        ref = torch.zeros(n, d_llm, device="cuda")
        for (j, src, dst_rank, dst_row, rows) in o["pieces"]:
            q = int(o["group"][j])
            x = torch.from_numpy(odp.standin(int(t["ids"][j]), int(t["lens"][j]), d_enc[q])
                                 .view(np.int16)).view(torch.bfloat16).cuda()
            off = src - int(o["enc_off"][j])
            ref[dst_row:dst_row + rows] = x[off:off + rows].float() @ Ws[q].float().t()
        err = (got - ref).abs()
        assert bool((err <= RTOL * ref.abs() + ATOL).all()), f"graph step {i}"
