"""Failure path of the cross-GPU exchange on one GPU (SURVEY §5 failure detection):
a flag wait that times out poisons the path's status word; a poisoned copy or
projector GEMM moves nothing and publishes its epoch with MUX_POISON_BIT; a
wait that sees that bit poisons its own path; later waits return at once; and
MuxPath.run_pipeline raises at its next call.  Every wait here is bounded and
depends on no other kernel (one GPU, no peer)."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import planner as oplan
from paper_2605_08962_b200 import _lib, planner
from paper_2605_08962_b200.dataplane import MuxPath
from tests.helpers import random_table
from tests.test_gpu_planner import to_table

pytestmark = pytest.mark.gpu

POISON = 1 << 63


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _wait(flags, epoch, err, timeout_ms):
    L = _lib.lib()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(L.mux_wait(1, flags.data_ptr(), epoch.data_ptr(), timeout_ms, err.data_ptr(),
                          _s()), "mux_wait")
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def test_wait_timeout_poisons_and_later_waits_fail_fast(cuda_device):
    flags = torch.zeros(1, dtype=torch.int64, device="cuda")
    epoch = torch.full((1,), 5, dtype=torch.int64, device="cuda")  # never reached
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ms = _wait(flags, epoch, err, 20)
    assert int(err.item()) == 1 and ms >= 15
    ms2 = _wait(flags, epoch, err, 20000)  # poisoned: returns at once
    assert int(err.item()) == 1 and ms2 < 5


def test_poison_bit_propagates_to_the_waiter(cuda_device):
    flags = torch.tensor([7 | POISON - (1 << 64)], dtype=torch.int64, device="cuda")
    epoch = torch.full((1,), 7, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _wait(flags, epoch, err, 20000)
    assert int(err.item()) == 2


def _plan(seed=3):
    rs = np.random.RandomState(seed)
    t, cap = random_table(rs, S=60, n_chunks=2, cap=256, n_carry_seqs=1)
    o = oplan.plan_step(t, cap, 2, 1, 1, 1)
    return t, cap, o


def test_poisoned_copy_moves_nothing_and_publishes_poison(cuda_device):
    t, cap, o = _plan()
    path = MuxPath(capacity=cap, gbs=2, dp=1, d_in=(16, 8), d_llm=64)
    table = to_table(t)
    plan = path.plan(planner.DeviceTable(table, "cuda"))
    plan.check(table)
    arenas = [torch.randn(max(int(o["arena_rows"][0, g]), 1), (16, 8)[g],
                          device="cuda").to(torch.bfloat16) for g in range(2)]
    for g in range(2):
        path.recv[g].tensor.fill_(0x5a)
    flags = torch.zeros(1, dtype=torch.int64, device="cuda")
    fptrs = torch.tensor([flags.data_ptr()], dtype=torch.int64, device="cuda")
    epoch = torch.zeros(1, dtype=torch.int64, device="cuda")
    sync = torch.zeros(2, dtype=torch.int32, device="cuda")
    L = _lib.lib()
    for poisoned in (False, True):
        err = torch.full((1,), int(poisoned), dtype=torch.int32, device="cuda")
        _lib.check(L.mux_segcopy_ex(C.byref(plan.cfg), plan.ptr, 0,
                                    path._arena_table(arenas).data_ptr(), path.recv_dst.data_ptr(),
                                    0, -1, fptrs.data_ptr(), sync.data_ptr(), epoch.data_ptr(),
                                    err.data_ptr(), _s()), "mux_segcopy_ex")
        torch.cuda.synchronize()
        f = int(flags.item()) & ((1 << 64) - 1)
        if not poisoned:  # the healthy copy moved the rows and published epoch 1
            assert f == 1
            n = int(o["recv_rows"][0, 0])
            assert torch.equal(path.recv_view(0, n).cpu(), arenas[0][:n].cpu()) or n == 0
            for g in range(2):
                path.recv[g].tensor.fill_(0x5a)
        else:  # nothing moved, epoch 2 with the poison bit
            assert f == (2 | POISON)
            for g in range(2):
                assert bool((path.recv[g].tensor == 0x5a).all())
    assert int(sync.sum().item()) == 0  # counters re-armed either way


def test_poisoned_projector_computes_nothing(cuda_device):
    M, K, N = 300, 128, 256
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = torch.full((M, N), 3.0, device="cuda").to(torch.bfloat16)
    rows = torch.arange(M, dtype=torch.int64, device="cuda")
    bases = torch.tensor([out.data_ptr()], dtype=torch.int64, device="cuda")
    flags = torch.zeros(1, dtype=torch.int64, device="cuda")
    fptrs = torch.tensor([flags.data_ptr()], dtype=torch.int64, device="cuda")
    epoch = torch.zeros(1, dtype=torch.int64, device="cuda")
    sync = torch.zeros(1, dtype=torch.int32, device="cuda")
    err = torch.ones(1, dtype=torch.int32, device="cuda")
    g = _lib.ProjGroup(X.data_ptr(), W.data_ptr(), 0, M, 0, K, 0, rows.data_ptr())
    arr = (_lib.ProjGroup * 1)(g)
    L = _lib.lib()
    _lib.check(L.mux_proj_scatter_grouped_signal(arr, 1, N, bases.data_ptr(), 0, 0, 1,
                                                 fptrs.data_ptr(), sync.data_ptr(),
                                                 epoch.data_ptr(), None, None, err.data_ptr(),
                                                 _s()), "proj")
    torch.cuda.synchronize()
    assert bool((out.float() == 3.0).all())
    assert (int(flags.item()) & ((1 << 64) - 1)) == (1 | POISON)
    err.zero_()  # healthy launch: computes and publishes epoch 2 without the bit
    _lib.check(L.mux_proj_scatter_grouped_signal(arr, 1, N, bases.data_ptr(), 0, 0, 1,
                                                 fptrs.data_ptr(), sync.data_ptr(),
                                                 epoch.data_ptr(), None, None, err.data_ptr(),
                                                 _s()), "proj")
    torch.cuda.synchronize()
    ref = X.float() @ W.float().t()
    assert bool(((out.float() - ref).abs() <= 2.0 ** -7 * ref.abs() + 1e-3 * K).all())
    assert int(flags.item()) == 2


def test_run_pipeline_raises_on_a_poisoned_path(cuda_device):
    """The host side: run_pipeline mirrors the status word asynchronously and
    raises at its next call; check_wait() raises after a sync."""
    t, cap, o = _plan(5)
    path = MuxPath(capacity=cap, gbs=2, dp=1, d_in=(16, 8), d_llm=64)
    table = to_table(t)
    dtab = planner.DeviceTable(table, "cuda")
    arenas = [torch.randn(max(int(o["arena_rows"][0, g]), 1), (16, 8)[g],
                          device="cuda").to(torch.bfloat16) for g in range(2)]
    # world 1 has no waits: emulate the mirror the multi-GPU path keeps
    path._status_host = torch.zeros(1, dtype=torch.int32).pin_memory()
    path.run_pipeline([(dtab, arenas)])
    torch.cuda.synchronize()
    path.run_pipeline([(dtab, arenas)])  # healthy: no raise
    path.wait_err.fill_(1)
    path.run_pipeline([(dtab, arenas)])  # the mirror of this call sees the poison
    torch.cuda.synchronize()
    with pytest.raises(RuntimeError, match="poisoned"):
        path.run_pipeline([(dtab, arenas)])
    with pytest.raises(RuntimeError, match="timed out"):
        path.check_wait()
