"""Encoder-rank balancing (reference module `muxsim.balance`).

The reference ships this module only as a specification.  Here every
partition runs on the GPU (libmuxb200 `mux_assign`, the same device code the
step planner uses):

* ``kk_partition``   g-way Karmarkar-Karp largest differencing;
                     the tuple-merge reading is pinned in DESIGN.md §KK.
* ``lpt_partition``  longest-processing-time greedy, the north_star's
                     "greedy/LPT" (BASELINE.json).
* ``grouped_reorder`` / ``restore_order``  pooled reorder within a group of
                     ranks with an exact inverse.
* ``zero_redundancy_filter``  which encoder microbatches a PP stage's loader
                     fetches.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib
from .planner import _stream_ptr
from .workload import GlobalBatch, Sample


def _assign(method: int, weights, g: int, ids=None, init=None) -> list[int]:
    if g < 1:
        raise ValueError("g must be >= 1")
    w = np.asarray(list(weights), dtype=np.float64)
    if w.size == 0:
        raise ValueError("weights must be nonempty")
    if (w < 0).any():
        raise ValueError("weights must be nonnegative")
    dev = torch.device("cuda", torch.cuda.current_device())
    wd = torch.from_numpy(w).to(dev)
    idd = torch.from_numpy(np.asarray(ids if ids is not None else np.arange(w.size),
                                      dtype=np.int64)).to(dev)
    out = torch.empty(w.size, dtype=torch.int32, device=dev)
    ini = None
    if init is not None:
        ini = torch.tensor([float(x) for x in init], dtype=torch.float64, device=dev)
        if ini.numel() != g:
            raise ValueError("init must hold one load per group")
    _lib.check(_lib.lib().mux_assign(method, wd.data_ptr(), idd.data_ptr(), int(w.size), int(g),
                                     out.data_ptr(), None if ini is None else ini.data_ptr(),
                                     _stream_ptr()), "mux_assign")
    return out.cpu().tolist()


def kk_partition(weights, g: int) -> list[int]:
    """Assignment weight index -> group of a g-way Karmarkar-Karp partition.

    Deterministic; ties break to the lower index; g > len(weights) leaves
    empty groups.
    """
    return _assign(_lib.KK, weights, g)


def lpt_partition(weights, g: int, ids=None, init=None) -> list[int]:
    """Greedy LPT: heaviest first (ties by id, then index) to the least-loaded rank;
    `init`: loads the g ranks start with."""
    return _assign(_lib.LPT, weights, g, ids, init)


@dataclass
class ReorderGroup:
    """Member ranks of one network-local group and their per-rank sample lists
    before reordering."""

    ranks: list[int]
    samples: list[list[Sample]]


@dataclass
class ReorderRecord:
    """Permutation record: (origin_rank, origin_pos) -> (rank, position)."""

    forward: dict[tuple[int, int], tuple[int, int]] = field(default_factory=dict)
    shape: list[int] = field(default_factory=list)   # pre-reorder list length per rank


def grouped_reorder(group: ReorderGroup, microbatch_window: int = 1, method: str = "kk"):
    """Pool the group's samples, partition by token count over the group's ranks,
    and return (balanced per-rank lists, record).

    Samples keep their (origin_rank, origin_pos); unassigned ones get (rank
    index in group, list position) as the loader would at load time
    (SPEC.md:51).  Within a destination rank, samples are ordered by
    (origin rank, origin position) — the natural all-to-allv receive order.
    Like the reference's operations, the caller's Samples are not mutated:
    the returned lists hold copies carrying their origin fields.
    """
    if microbatch_window < 1:
        raise ValueError("microbatch_window must be >= 1")
    pool: list[Sample] = []
    shape = []
    for r, lst in enumerate(group.samples):
        shape.append(len(lst))
        for pos, s in enumerate(lst):
            if s.origin_rank < 0:
                s = replace(s, origin_rank=r, origin_pos=pos)
            else:
                s = replace(s)
            pool.append(s)
    g = len(group.ranks)
    out: list[list[Sample]] = [[] for _ in range(g)]
    rec = ReorderRecord(shape=shape)
    if not pool:
        return out, rec
    w = [s.length for s in pool]
    if method == "kk":
        assign = kk_partition(w, g)
    elif method == "lpt":
        assign = lpt_partition(w, g, ids=[s.id for s in pool])
    else:
        raise ValueError(f"unknown method {method!r}")
    for s, r in sorted(zip(pool, assign), key=lambda t: (t[0].origin_rank, t[0].origin_pos)):
        rec.forward[(s.origin_rank, s.origin_pos)] = (r, len(out[r]))
        out[r].append(s)
    return out, rec


def restore_order(record: ReorderRecord, reordered: list[list] | None = None):
    """Exact inverse of grouped_reorder.

    With `reordered` (per-rank lists in reordered positions — samples,
    embeddings or gradients), returns them in original per-rank order.
    Without it, returns the inverse map (rank, pos) -> (origin_rank, origin_pos).
    Raises ValueError on a corrupted record.
    """
    inverse = {v: k for k, v in record.forward.items()}
    if len(inverse) != len(record.forward):
        raise ValueError("corrupted reorder record: duplicate destinations")
    if reordered is None:
        return inverse
    out = [[None] * n for n in record.shape]
    for (r, p), (orank, opos) in inverse.items():
        try:
            out[orank][opos] = reordered[r][p]
        except IndexError as e:
            raise ValueError("corrupted reorder record") from e
    if any(x is None for lst in out for x in lst):
        raise ValueError("corrupted reorder record: missing entries")
    return out


def zero_redundancy_filter(batch: GlobalBatch, stage: int, pp: int,
                           n_encoder_microbatches: int | None = None) -> list[int]:
    """Encoder microbatch indices stage `stage` of a pp-stage pipeline fetches
    under the uniform insertion rule: {stage, stage+pp, ...}."""
    if not 0 <= stage < pp:
        raise ValueError(f"stage {stage} outside 0..{pp - 1}")
    n = n_encoder_microbatches
    if n is None:
        n = batch.microbatches_per_replica * batch.dp_degree
    return list(range(stage, n, pp))


def imbalance(loads) -> float:
    """max / mean load (SPEC.md:405 reports 10/3.25 for [10,1,1,1])."""
    a = np.asarray(loads, dtype=np.float64)
    return float(a.max() / a.mean()) if a.size and a.mean() > 0 else 1.0


def loads_of(weights, assign, g: int) -> list[float]:
    return np.bincount(np.asarray(assign), weights=np.asarray(weights, np.float64),
                       minlength=g).tolist()
