"""Regenerate the golden vectors from the REFERENCE implementation.

Runs only in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports the reference's own `muxsim.workload` (PEP 420 namespace package
under /root/reference/pkg/src) and records what the
reference produces on fixed seeds and on hand-made edge cases.  The JSON files
it writes are committed; the tests and the GPU box only read them.
numpy version used is stored in each file (the RNG stream is numpy's PCG64).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")

import muxsim.workload as ref  # noqa: E402  (the reference itself)

from paper_2605_08962_b200 import configs  # noqa: E402


def _samples(lst):
    return [[s.id, s.modality.value, s.dataset, s.length] for s in lst]


def _seqs(lst):
    return [[list(sp) for sp in q.spans] for q in lst]


def _dump(name, obj):
    obj["numpy"] = np.__version__
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print("wrote", name)


def gen_configs():
    """Chained generate_batch steps per config (workload.py:281-305)."""
    out = {}
    for name, cfg in configs.CONFIGS.items():
        reg, sched = configs.build(ref, name)
        if cfg["gbs_per_replica"] is None:
            chunk = ref.sample_step(reg, sched, 0, cfg["toy_n"], cfg["seed"])
            out[name] = dict(toy=True, samples=_samples(chunk),
                             seqs=_seqs(ref.hybrid_pack(chunk, configs.CAPACITY)))
            continue
        steps = []
        for world in (1, 2, 8) if name in ("cfg3", "cfg5") else (1,):
            carry = None
            dp = world if cfg["sp"] == 1 else 2
            if name == "cfg4":
                world, dp = 8, 2
            gbs = cfg["gbs_per_replica"] * dp
            for step in range(3):
                drawn = []
                batch, rest = ref.generate_batch(
                    reg, sched, step, cfg["seed"], gbs, dp, 1, configs.CAPACITY,
                    carry if cfg["carry"] else None, drawn)
                steps.append(dict(world=world, dp=dp, gbs=gbs, step=step,
                                  carry_in=_seqs(carry or []) if cfg["carry"] else [],
                                  drawn=_samples(drawn),
                                  batch=_seqs(batch.sequences),
                                  carry_out=_seqs(rest)))
                carry = rest
            if name == "cfg4":
                break
        out[name] = dict(toy=False, steps=steps)
    _dump("configs.json", out)


def gen_pack_cases():
    """hybrid_pack on random and hand-made inputs (workload.py:240-262)."""
    rs = np.random.RandomState(20260518)
    cases = []
    for k in range(60):
        n = int(rs.randint(0, 300))
        cap = int(rs.choice([16, 100, 1000, 16384]))
        hi = cap if k % 3 else max(cap // 4, 1)
        lens = rs.randint(0 if k % 5 == 0 else 1, hi + 1, size=n).tolist()
        if k % 4 == 0:   # many duplicate ids: stable order must survive
            ids = rs.randint(0, max(n // 3, 1), size=n).tolist()
        else:
            ids = rs.permutation(n).tolist()
        samples = [ref.Sample(id=i, modality=ref.Modality.IMAGE, dataset="x", length=L)
                   for i, L in zip(ids, lens)]
        cases.append(dict(cap=cap, ids=ids, lens=lens,
                          seqs=_seqs(ref.hybrid_pack(samples, cap))))
    # SPEC.md:85-87 known answers, zero-length into a full bin, oversize error.
    hand = [
        ([9, 7, 5, 3, 2], 16), ([16], 16), ([1] * 48, 16), ([], 16),
        ([16, 0, 16, 0], 16), ([5, 0, 11, 0, 3], 16),
    ]
    for lens, cap in hand:
        samples = [ref.Sample(id=i, modality=ref.Modality.TEXT, dataset="x", length=L)
                   for i, L in enumerate(lens)]
        cases.append(dict(cap=cap, ids=list(range(len(lens))), lens=lens,
                          seqs=_seqs(ref.hybrid_pack(samples, cap))))
    errors = []
    for ids, lens, cap in (([3, 7, 1, 9], [4, 20, 5, 30], 16),
                           ([9, 7], [30, 20], 16), ([5], [17], 16)):
        samples = [ref.Sample(id=i, modality=ref.Modality.AUDIO, dataset="x", length=L)
                   for i, L in zip(ids, lens)]
        try:
            ref.hybrid_pack(samples, cap)
            msg = None
        except ref.PackingError as e:
            msg = str(e)
        errors.append(dict(ids=ids, lens=lens, cap=cap, message=msg))
    _dump("pack_cases.json", dict(cases=cases, errors=errors))


def gen_misc():
    """recipe_at / build_global_batch known answers."""
    mix0 = ref.MixtureRecipe.of(image=0.5, text=0.5)
    mix1 = ref.MixtureRecipe.of(image=0.13, audio=0.74, text=0.13)
    lin = ref.PhaseSchedule(((0, mix0), (1000, mix1)), ref.Interpolation.LINEAR)
    recipes = {str(s): [list(e) for e in lin.recipe_at(s).entries]
               for s in (0, 1, 250, 500, 999, 1000, 5000)}
    gb = []
    for n, gbs, dp, mbs in ((8, 8, 2, 1), (10, 8, 2, 1), (8, 8, 3, 1), (5, 8, 2, 1),
                            (5, 8, 3, 1), (12, 12, 3, 2)):
        seqs = [ref.PackedSequence(16, [(i, i + 1)]) for i in range(n)]
        try:
            b, rest = ref.build_global_batch(seqs, 0, gbs, dp, mbs)
            res = dict(batch=len(b.sequences), carry=len(rest),
                       mbs_per_replica=b.microbatches_per_replica,
                       replica_mb=[[[sp[0] for q in b.replica_microbatch(r, m) for sp in q.spans]
                                    for m in range(b.microbatches_per_replica)]
                                   for r in range(dp)])
        except ref.ConfigError as e:
            res = dict(error="ConfigError", message=str(e))
        except ValueError as e:
            res = dict(error="ValueError", message=str(e))
        gb.append(dict(n=n, gbs=gbs, dp=dp, mbs=mbs, result=res))
    _dump("misc.json", dict(recipes=recipes, build_global_batch=gb))


def gen_export():
    """export_batch (workload.py:308-324) of two chained cfg5 steps at dp=8: the
    reference's JSONL bytes, with the batch and the sample map that made them."""
    import tempfile
    reg, sched = configs.build(ref, "cfg5")
    cfg = configs.CONFIGS["cfg5"]
    carry, recs = None, []
    for step in range(2):
        drawn = []
        batch, carry_next = ref.generate_batch(reg, sched, step, cfg["seed"], 16, 8, 1,
                                               configs.CAPACITY, carry, drawn)
        samples = {s.id: s for s in drawn}
        with tempfile.NamedTemporaryFile("r", suffix=".jsonl") as fh:
            ref.export_batch(batch, samples, fh.name)
            text = open(fh.name).read()
        recs.append(dict(step=step, dp=8, mbs=1, capacity=configs.CAPACITY,
                         seqs=_seqs(batch.sequences), samples=_samples(drawn), jsonl=text))
        carry = carry_next
    _dump("export.json", dict(batches=recs))


if __name__ == "__main__":
    gen_configs()
    gen_pack_cases()
    gen_misc()
    gen_export()
