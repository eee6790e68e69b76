"""The multi-rank data plane emulated on ONE GPU: every rank's own device plan
(cfg.me = r) drives the same copy kernel, with the other ranks' receive windows
and LLM buffers standing in for NVLink peers (plain device pointers in the
per-rank pointer tables).  No cross-rank flags are used, so no kernel waits on
another (B200_PROFILING.md: never emulate waiting ranks as separate launches).
This runs the 2-, 4- and 8-rank dispatch / return / gradient tables of the
golden steps bit-exactly against the oracle on a one-GPU box — the protocol's
flag handshake is covered by tests/test_gpu_multi.py and the gloo tests."""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import dataplane as odp
from oracle import planner as oplan
from paper_2605_08962_b200 import _lib, configs, planner
from tests.helpers import golden_steps, random_table
from tests.test_gpu_planner import to_table

pytestmark = pytest.mark.gpu
G = _lib.N_GROUPS


def _tab(ptrs):
    return torch.tensor([int(p) for p in ptrs], dtype=torch.int64, device="cuda")


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def emulate(t, cap, gbs, dp, sp, world, method, d_in=(20, 12), d_llm=24, seed=11):
    """Every rank's plan, dispatch, stand-in encoder, return and gradient return on
    one GPU; returns nothing, asserts bit-exactness against the oracle."""
    L = _lib.lib()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    o = oplan.plan_step(t, cap, gbs, dp, sp, world, 1, method)
    table = to_table(t)
    dtab = planner.DeviceTable(table, "cuda")
    g0 = torch.Generator().manual_seed(seed)
    arenas = [[torch.randn(max(int(o["arena_rows"][r, g]), 1), d_in[g], generator=g0)
               .to(torch.bfloat16).cuda() for g in range(G)] for r in range(world)]
    recv = [[torch.zeros(max(int(o["recv_rows"][r, g]), 1), d_in[g], dtype=torch.bfloat16,
                         device="cuda") for g in range(G)] for r in range(world)]
    enc = [[torch.zeros(max(int(o["recv_rows"][r, g]), 1), d_llm, dtype=torch.bfloat16,
                        device="cuda") for g in range(G)] for r in range(world)]
    llm = [torch.zeros(max(int(o["llm_rows"][r]), 1), d_llm, dtype=torch.bfloat16,
                       device="cuda") for r in range(world)]
    grad = [[torch.zeros(max(int(o["recv_rows"][r, g]), 1), d_llm, dtype=torch.bfloat16,
                         device="cuda") for g in range(G)] for r in range(world)]
    dys = [torch.randn(max(int(o["llm_rows"][r]), 1), d_llm, generator=g0)
           .to(torch.bfloat16).cuda() for r in range(world)]
    recv_dst = _tab([recv[r][g].data_ptr() for r in range(world) for g in range(G)])
    llm_dst = _tab([x.data_ptr() for x in llm])
    grad_dst = _tab([grad[r][g].data_ptr() for r in range(world) for g in range(G)])
    sync = torch.zeros(8, dtype=torch.int32, device="cuda")
    plans = []
    for r in range(world):  # every rank plans the whole step itself
        cfg = planner.make_cfg(table, cap, gbs, dp, sp, world, 1, method, False, r,
                               row_bytes_in=tuple(2 * d for d in d_in),
                               row_bytes_ret=(2 * d_llm,) * G, row_bytes_grad=(2 * d_llm,) * G)
        p = planner.plan_step(dtab, cfg)
        p.check(table)
        plans.append(p)
    for r in range(world):  # dispatch: rank r's arena rows to every encoder rank
        _lib.check(L.mux_segcopy(C.byref(plans[r].cfg), plans[r].ptr, 0,
                                 _tab([a.data_ptr() for a in arenas[r]]).data_ptr(),
                                 recv_dst.data_ptr(), 0, sync[0:].data_ptr(), s))
    for r in range(world):  # encoder stand-in on every rank
        for g in range(G):
            _lib.check(L.mux_encoder_standin(C.byref(plans[r].cfg), plans[r].ptr, dtab.ids,
                                             dtab.lens, g, d_llm, enc[r][g].data_ptr(), s))
    for r in range(world):  # return: rank r's encoder rows to their LLM ranks
        _lib.check(L.mux_segcopy(C.byref(plans[r].cfg), plans[r].ptr, 1,
                                 _tab([e.data_ptr() for e in enc[r]]).data_ptr(),
                                 llm_dst.data_ptr(), 0, sync[2:].data_ptr(), s))
    for r in range(world):  # gradient return: rank r's dY rows to the encoder ranks
        _lib.check(L.mux_segcopy(C.byref(plans[r].cfg), plans[r].ptr, 2,
                                 _tab([dys[r].data_ptr()] * G).data_ptr(),
                                 grad_dst.data_ptr(), 0, sync[4:].data_ptr(), s))
    torch.cuda.synchronize()
    ar = [[_bits(a) for a in arenas[r]] for r in range(world)]
    want_recv, _, want_llm = odp.run_world(o, t, world, ar, d_in, (d_llm,) * G, d_llm)
    want_grad = odp.run_grad(o, world, [_bits(d) for d in dys], d_llm)
    for r in range(world):
        for g in range(G):
            k = int(o["recv_rows"][r, g])
            assert np.array_equal(_bits(recv[r][g])[:k], want_recv[r][g]), (r, g)
            assert np.array_equal(_bits(grad[r][g])[:k], want_grad[r][g]), (r, g)
        k = int(o["llm_rows"][r])
        assert np.array_equal(_bits(llm[r])[:k], want_llm[r]), r


@pytest.mark.parametrize("method", ["lpt", "lpt_local"])
def test_emulated_world_matches_oracle(cuda_device, method):
    n = 0
    for name, st, t, _ in golden_steps():
        world, dp = st["world"], st["dp"]
        if world < 2 or st["step"] > 1:
            continue
        emulate(t, configs.CAPACITY, st["gbs"], dp, world // dp, world, method)
        n += 1
    assert n >= 4


def test_emulated_world_random_tables(cuda_device):
    """Edge cases of the reference's tests, across 2/4/8 emulated ranks: zero-length
    samples, duplicate ids, text-only samples, carried sequences, tiny capacities,
    Ulysses sp > 1 — every rank's buffers bit-exact."""
    rs = np.random.RandomState(23)
    done = 0
    for it in range(30):
        t, cap = random_table(rs)
        world, dp = [(2, 2), (2, 1), (4, 4), (4, 2), (8, 8), (8, 2)][it % 6]
        gbs = dp * int(rs.randint(1, 3))
        try:
            oplan.plan_step(t, cap, gbs, dp, world // dp, world, 1, "lpt_local")
        except ValueError:
            continue  # not enough sequences / oversize: the planner's error paths
        emulate(t, cap, gbs, dp, world // dp, world, ("lpt", "lpt_local", "kk")[it % 3],
                seed=it)
        done += 1
    assert done >= 10
