"""CpHybrid LLM placement on the data path — TEST INFRASTRUCTURE ONLY (CPU restatement).

reshard.plan_reshard's CpHybrid variant (
PAPER.md §5.2 "only shard long samples") applied to a step plan: within each
batch sequence's CP group (the replica's cp = sp ranks), samples longer than
cp_threshold (default capacity / cp) are split cp ways with the
Ulysses rule (first L mod cp pieces one token longer); the others stay whole
and go to a rank by LPT whose initial loads are the long-sample pieces
(the SPEC's "kk_partition on residual capacity" is
ill-defined for KK).  This is oracle/planner.py plan_reshard's cp_hybrid
branch, indexed by span position instead of sample id.

Pinned data layout: on CP rank k of replica r, the rows
of sequence q are q's pieces that rank k holds, in span order; sequences of
the replica follow each other in batch order.  Every LLM token, text
included, has a row.  The encoder side is unchanged; only the return pieces,
the LLM row counts and the per-(sequence, rank) loads change.  The GPU's
segment copies then push every encoder row straight to its CP rank (the
SPEC's all-reduce "dispatch primitive" models the same placement as a
collective; here it is one hop of point-to-point stores).
"""

from __future__ import annotations

import numpy as np

from .lssp import shard
from .planner import lpt_assign


def place(plan: dict, table: dict, gbs: int, dp: int, cp: int, capacity: int,
          cp_threshold: int | None = None) -> dict:
    """Copy of `plan` with CpHybrid pieces, row_base, llm_rows and loads."""
    lens = np.asarray(table["lens"], np.int64)
    ids = np.asarray(table["ids"], np.int64)
    thr = cp_threshold if cp_threshold else capacity // cp
    P = gbs // dp
    seq, span = plan["seq"], plan["span"]
    members = {}
    for i in range(len(lens)):
        if 0 <= seq[i] < gbs:
            members.setdefault(int(seq[i]), []).append(i)
    load = np.zeros((gbs, cp), np.int64)
    local = {}          # i -> list of (k, t0, n, local row)
    for q in range(gbs):
        sp_list = sorted(members.get(q, []), key=lambda i: span[i])
        short = []
        rank_of = {}
        for i in sp_list:
            if lens[i] > thr:
                for k in range(cp):
                    load[q, k] += shard(lens[i], cp, k)[1]
            else:
                short.append(i)
        if short:
            ranks = lpt_assign([float(lens[i]) for i in short], [int(ids[i]) for i in short],
                               cp, init=[float(x) for x in load[q]])
            for i, r in zip(short, ranks):
                rank_of[i] = r
                load[q, r] += lens[i]
        off = [0] * cp
        for i in sp_list:
            if lens[i] > thr:
                pcs = []
                for k in range(cp):
                    s0, n = shard(lens[i], cp, k)
                    pcs.append((k, s0, n, off[k]))
                    off[k] += n
                local[i] = pcs
            else:
                r = rank_of[i]
                local[i] = [(r, 0, int(lens[i]), off[r])]
                off[r] += int(lens[i])
    row_base = np.zeros((gbs, cp), np.int64)
    world = dp * cp
    llm_rows = np.zeros(world, np.int64)
    for q in range(gbs):
        r = q // P
        for k in range(cp):
            row_base[q, k] = llm_rows[r * cp + k]
            llm_rows[r * cp + k] += load[q, k]
    pieces = []
    for i in np.flatnonzero(plan["enc"] >= 0).tolist():   # table order
        q = int(seq[i])
        for (k, t0, n, lrow) in local[i]:
            if n > 0:
                pieces.append((i, int(plan["enc_off"][i]) + t0, (q // P) * cp + k,
                               int(row_base[q, k]) + lrow, n))
    text_pieces = []
    for i in range(len(lens)):
        if 0 <= seq[i] < gbs and plan["group"][i] < 0:
            q = int(seq[i])
            for (k, t0, n, lrow) in local[i]:
                if n > 0:
                    text_pieces.append((i, t0, (q // P) * cp + k, int(row_base[q, k]) + lrow, n))
    out = dict(plan)
    out.update(pieces=pieces, text_pieces=text_pieces, llm_rows=llm_rows, row_base=row_base,
               shard_len=load, cp_threshold=thr)
    return out
