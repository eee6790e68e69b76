"""The multi-rank protocol on CPU (gloo, world size 2): every rank plans the
whole step on its own, derives its own segment tables, pushes its rows, and the
ranks end up with exactly the oracle's per-rank buffers — with no counts
exchanged.  This is the host-side logic of the NVLink push exchange; the GPU
tests run the same protocol with the CUDA kernels (tests/mgpu_worker.py)."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dataplane as odp
from oracle import planner as oplan
from tests.helpers import golden_steps


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _digest(plan):
    h = hashlib.sha256()
    for k in ("seq", "off", "origin", "enc", "arena_off", "enc_off", "recv_rows", "llm_rows"):
        h.update(np.ascontiguousarray(plan[k]).tobytes())
    h.update(repr(plan["pieces"]).encode())
    return h.hexdigest()


def _worker(rank, world, port, cases, result_q, mode="plain"):
    from oracle import cphybrid as ocph
    from oracle import lssp as olssp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    for t, st, d_in, d_llm in cases:
        plan = oplan.plan_step(t, 16384, st["gbs"], st["dp"], world // st["dp"], world)
        if mode == "cp":
            plan = ocph.place(plan, t, st["gbs"], st["dp"], world // st["dp"], 16384, 2048)
        lay = olssp.layout(plan, t["lens"], world, 2048, world) if mode == "lssp" else None
        digests = [None] * world
        dist.all_gather_object(digests, _digest(plan))
        ok &= len(set(digests)) == 1  # every rank computed the identical plan
        # every rank's loader arena is seeded, so the oracle can rebuild all ranks
        g = np.random.default_rng(7)
        arenas = [[g.integers(0, 2 ** 16, size=(int(plan["arena_rows"][r, q]), d_in[q]),
                              dtype=np.uint16) for q in range(2)] for r in range(world)]
        # dispatch: my segments, pushed as (dst rank, group, dst row, rows payload)
        sends = [[] for _ in range(world)]
        dsegs = odp.dispatch_by_rank(plan, t["lens"], rank) if lay is None else \
            olssp.dispatch_by_rank(plan, lay, t["lens"], rank)
        for src, dst, n, q, to in dsegs.tolist():
            sends[to].append((q, dst, arenas[rank][q][src:src + n]))
        got = [None] * world
        dist.all_gather_object(got, sends)
        rows_of = plan["recv_rows"] if lay is None else lay["recv_rows"]
        recv = [np.zeros((int(rows_of[rank, q]), d_in[q]), np.uint16) for q in range(2)]
        for r in range(world):
            for q, dst, rows in got[r][rank]:
                recv[q][dst:dst + len(rows)] = rows
        if lay is None:
            ref_recv, enc_out, ref_llm = odp.run_world(plan, t, world, arenas, d_in,
                                                       (d_llm,) * 2, d_llm)
        else:
            ref_recv, enc_out, ref_llm = olssp.run_world(plan, lay, t, world, arenas, d_in,
                                                         (d_llm,) * 2, d_llm)
        ok &= all(np.array_equal(recv[q], ref_recv[rank][q]) for q in range(2))
        # return: my encoder rows to their LLM ranks
        sends = [[] for _ in range(world)]
        rsegs = odp.pieces_by_rank(plan, rank) if lay is None else olssp.return_by_rank(lay, rank)
        for src, dst, n, q, to in rsegs.tolist():
            sends[to].append((dst, enc_out[rank][q][src:src + n]))
        got = [None] * world
        dist.all_gather_object(got, sends)
        llm = np.zeros((int(plan["llm_rows"][rank]), d_llm), np.uint16)
        for r in range(world):
            for dst, rows in got[r][rank]:
                llm[dst:dst + len(rows)] = rows
        ok &= np.array_equal(llm, ref_llm[rank])
    result_q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "plain"), (2, "lssp"), (2, "cp")])
def test_push_protocol_gloo(world, mode):
    """Plain Ulysses placement, the LSSP eta split (group = both ranks, eta 2048)
    and CpHybrid placement (threshold 2048): each rank's segment tables alone
    rebuild every buffer."""
    cases = []
    for name, st, t, _ in golden_steps():
        if st["world"] == world and name in ("cfg5", "cfg3") and st["step"] < 2:
            if mode == "cp" and st["dp"] == world:
                st = dict(st, dp=1)  # one replica, its CP group = both ranks
            cases.append((t, st, (12, 4), 16))
    assert cases
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q, mode))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}


def _meta_worker(rank, world, port, cases, result_q):
    """Decentralized loaders: each rank packs only its share of the step into a
    metadata record; one all-gather (gloo here, NCCL on the GPUs) and the
    record assembly rebuild the global table on every rank, so every rank's
    plan equals the centralized one."""
    from paper_2605_08962_b200 import planner
    from tests.test_gpu_planner import to_table
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    cap, capc = 1024, 32
    for t, st in cases:
        table = to_table(t)
        rec = torch.from_numpy(table.shard(rank, world).record(cap, capc))
        out = [torch.empty_like(rec) for _ in range(world)]
        dist.all_gather(out, rec)
        got = oplan.assemble_records([o.numpy() for o in out], cap, capc)
        for k in ("lens", "mods", "ids", "carry_seq"):
            ok &= np.array_equal(got[k], np.asarray(t[k]))
        ok &= list(got["chunk_off"]) == list(t["chunk_off"])
        ok &= got["n_carry_seqs"] == t["n_carry_seqs"]
        a = oplan.plan_step(got, 16384, st["gbs"], st["dp"], world // st["dp"], world)
        b = oplan.plan_step(t, 16384, st["gbs"], st["dp"], world // st["dp"], world)
        ok &= _digest(a) == _digest(b)
    result_q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_metadata_all_gather_gloo(world):
    cases = [(t, dict(st, dp=1)) for name, st, t, _ in golden_steps()
             if name in ("cfg5", "cfg4", "target1") and st["step"] < 2]
    assert cases
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_meta_worker, args=(r, world, port, cases, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}
