"""Encoder -> LLM resharding (reference module `muxsim.reshard`).

The reference ships this module only as a specification.  Here the shard
geometry comes from the device planner (libmuxb200 `mux_plan_step`: Ulysses
shard starts/lengths per sequence, the same arrays the return exchange uses)
and CpHybrid's short-sample placement from the device LPT with initial loads
(`mux_assign`).  The host only lists, per sample, the token ranges that fall
into each shard.

* ``plan_reshard``   UlyssesUniform (each sequence in sp equal shards, first
                     F mod sp shards one token longer) or CpHybrid
                     (long samples split cp-way, short ones whole, balanced on
                     residual capacity).
* ``dispatch_cost``  the modeled comparator of the exchange,
                     through costs.comm_time (pkg/src/muxsim/costs.py:95-105).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import costs
from .balance import lpt_partition
from .planner import DeviceTable, StepTable, make_cfg, plan_step
from .workload import PackedSequence


class ReshardVariant(str, Enum):
    ULYSSES_UNIFORM = "ulysses"
    CP_HYBRID = "cp_hybrid"


@dataclass
class ReshardPlan:
    variant: ReshardVariant
    shard_map: dict[int, list[tuple[int, int, int]]] = field(default_factory=dict)
    primitive: str = "all_to_all"
    tokens_per_rank: list[list[int]] = field(default_factory=list)  # per sequence
    degenerate: bool = False  # some shard holds no token (sequence shorter than sp)


def _degree(llm_layout, attr):
    if isinstance(llm_layout, int):
        return llm_layout
    return int(getattr(llm_layout, attr))


def plan_reshard(sequences: list[PackedSequence], llm_layout, variant, cp_threshold=None):
    """Shard map sample id -> [(rank, start, end)] over one SP/CP group.

    `llm_layout`: the group size (int) or an object with `.sp` (Ulysses) /
    `.cp` (CpHybrid).  Token ranges are contiguous, disjoint and cover each
    sample.
    """
    variant = ReshardVariant(variant)
    plan = ReshardPlan(variant=variant)
    if not sequences:
        return plan
    if variant == ReshardVariant.ULYSSES_UNIFORM:
        sp = _degree(llm_layout, "sp")
        if sp < 1:
            raise ValueError("sp must be >= 1")
        # device geometry: the sequences as one step's carried batch, dp=1, sp ranks
        lens, ids, cseq = [], [], []
        for q, seq in enumerate(sequences):
            for sid, tok in seq.spans:
                lens.append(tok)
                ids.append(sid)
                cseq.append(q)
        n = len(lens)
        table = StepTable(np.asarray(lens, np.int32), np.ones(n, np.int32),
                          np.asarray(ids, np.int64), np.asarray(cseq, np.int32), len(sequences),
                          np.asarray([n], np.int32))
        cap = max(max(s.capacity for s in sequences), 1)
        cfg = make_cfg(table, cap, gbs=len(sequences), dp=1, sp=sp, world=sp)
        dev = torch.device("cuda", torch.cuda.current_device())
        p = plan_step(DeviceTable(table, dev), cfg)
        p.check(table)
        h = p.host()
        starts = h["shard_start"].reshape(len(sequences), sp)
        slens = h["shard_len"].reshape(len(sequences), sp)
        for i in range(n):
            q, off, L = int(h["seq"][i]), int(h["off"][i]), int(lens[i])
            pieces = []
            for k in range(sp):
                a = max(off, int(starts[q, k]))
                b = min(off + L, int(starts[q, k]) + int(slens[q, k]))
                if a < b:
                    pieces.append((k, a - off, b - off))
            plan.shard_map[ids[i]] = pieces
        plan.tokens_per_rank = slens.tolist()
        plan.degenerate = bool((slens == 0).any())
        plan.primitive = "all_to_all"
        return plan
    cp = _degree(llm_layout, "cp")
    if cp < 1:
        raise ValueError("cp must be >= 1")
    thr = cp_threshold if cp_threshold is not None else \
        max(s.capacity for s in sequences) // cp
    if thr < 1:
        raise ValueError("cp_threshold must be >= 1")
    for seq in sequences:
        load = [0] * cp
        short = []
        for sid, tok in seq.spans:
            if tok > thr:
                q, r = divmod(tok, cp)
                off = 0
                plan.shard_map[sid] = []
                for k in range(cp):
                    n = q + (1 if k < r else 0)
                    plan.shard_map[sid].append((k, off, off + n))
                    load[k] += n
                    off += n
            else:
                short.append((sid, tok))
        if short:
            ranks = lpt_partition([t for _, t in short], cp, ids=[s for s, _ in short],
                                  init=load) if cp > 1 else [0] * len(short)
            for (sid, tok), r in zip(short, ranks):
                plan.shard_map[sid] = [(r, 0, tok)]
                load[r] += tok
        plan.tokens_per_rank.append(load)
    plan.primitive = "all_reduce"
    return plan


def dispatch_cost(plan: ReshardPlan, comm: costs.CommModel, bytes_per_token: int = 2 * 4096,
                  intra_node: bool = True):
    """Modeled cost of the reshard exchange: one symmetric
    all-to-all per UlyssesUniform sequence (per-rank payload = its shard),
    one all-reduce sized to the largest per-rank aggregate for CpHybrid.
    Returns (events, seconds); an empty plan costs nothing."""
    events, total = [], 0.0
    for loads in plan.tokens_per_rank:
        g = len(loads)
        nbytes = max(loads) * bytes_per_token
        t = costs.comm_time(comm, plan.primitive, nbytes, g, intra_node)
        events.append((plan.primitive, g, nbytes, t))
        total += t
    return events, total
