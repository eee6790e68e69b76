"""CPU restatement of the reference's synthetic generator and FFD packer.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
reference lines it restates; pinned against tests/golden/*.json, which
tests/golden/make_golden.py produced by running the reference itself.

Plain data shapes, independent of the product's classes:
  descriptor  dict(name, modality, mean, max_len, p95=0.0, hist=())
  recipe      list of (dataset, ratio), sorted by dataset name
  sample      tuple (id, modality, dataset, length)
  sequence    list of (sample id, tokens) spans
"""

from __future__ import annotations

import math

import numpy as np

Z95 = 1.6448536269514722  # workload.py:19


class OracleConfigError(ValueError):
    pass


class OraclePackingError(ValueError):
    pass


def lognormal_fit(mean: float, p95: float):
    """(mu, sigma) of a lognormal with the given mean and p95 (workload.py:54-65)."""
    target = p95 if p95 > 0 else 2.0 * mean
    spread = math.log(target / mean)
    if spread <= 0:
        return math.log(mean), 1e-6
    disc = Z95 * Z95 - 2.0 * spread
    if disc < 0:
        raise OracleConfigError("p95/mean ratio too large for a lognormal fit")
    sigma = Z95 - math.sqrt(disc)
    return math.log(mean) - 0.5 * sigma * sigma, sigma


def draw_lengths(desc: dict, rng, n: int) -> np.ndarray:
    """Length draws for one dataset (workload.py:67-78)."""
    hist = desc.get("hist", ())
    if hist:
        lo = np.array([h[0] for h in hist], dtype=np.float64)
        hi = np.array([h[1] for h in hist], dtype=np.float64)
        wt = np.array([h[2] for h in hist], dtype=np.float64)
        which = rng.choice(len(wt), size=n, p=wt / wt.sum())
        raw = lo[which] + rng.random(n) * (hi[which] - lo[which])
    else:
        mu, sigma = lognormal_fit(desc["mean"], desc.get("p95", 0.0))
        raw = rng.lognormal(mu, sigma, size=n)
    return np.clip(np.rint(raw), 1, desc["max_len"]).astype(np.int64)


def recipe_at(phases, step: int, linear: bool):
    """Recipe active at `step` (workload.py:121-137).  phases: [(start, {ds: r})]."""
    if step < 0:
        raise ValueError("step must be nonnegative")
    k = max(i for i, (start, _) in enumerate(phases) if start <= step)
    if not linear or k == len(phases) - 1:
        return sorted(phases[k][1].items())
    (s0, r0), (s1, r1) = phases[k], phases[k + 1]
    t = (step - s0) / (s1 - s0)
    names = sorted(set(r0) | set(r1))
    mixed = {nm: (1 - t) * r0.get(nm, 0.0) + t * r1.get(nm, 0.0) for nm in names}
    total = sum(mixed.values())
    return sorted((nm, v / total) for nm, v in mixed.items())


def draw_step(descs: dict, phases, linear: bool, step: int, n: int, seed: int,
              id_base: int = 0):
    """n samples for `step` (workload.py:209-237): dataset choice, then
    per-dataset lengths in alphabetical dataset order from one PCG64 stream."""
    if n < 1:
        raise ValueError("n must be >= 1")
    recipe = recipe_at(phases, step, linear)
    names = [nm for nm, _ in recipe]
    for nm in names:
        if nm not in descs:
            raise OracleConfigError(f"unknown dataset {nm!r}")
    p = np.array([r for _, r in recipe], dtype=np.float64)
    rng = np.random.default_rng(np.random.SeedSequence([seed, step]))
    pick = rng.choice(len(names), size=n, p=p / p.sum())
    out = [None] * n
    for k, nm in enumerate(names):
        where = np.flatnonzero(pick == k)
        if where.size:
            lens = draw_lengths(descs[nm], rng, where.size)
            for i, L in zip(where.tolist(), lens.tolist()):
                out[i] = (id_base + i, descs[nm]["modality"], nm, int(L))
    return out


def ffd(samples, capacity: int):
    """First-fit-decreasing across modalities (workload.py:240-262).

    Returns a list of sequences, each a list of (id, tokens) spans.  The
    oversize error names the first offender in input order (:245-248); the
    sort key is (-length, id) with Python's stable sort (:249); first fit
    scans bins in creation order (:252-261).
    """
    for s in samples:
        if s[3] > capacity:
            raise OraclePackingError(
                f"sample {s[0]} ({s[3]} tokens) exceeds capacity {capacity}")
    seqs, fills = [], []
    for s in sorted(samples, key=lambda t: (-t[3], t[0])):
        for b, f in enumerate(fills):
            if f + s[3] <= capacity:
                seqs[b].append((s[0], s[3]))
                fills[b] = f + s[3]
                break
        else:
            seqs.append([(s[0], s[3])])
            fills.append(s[3])
    return seqs


def take_batch(seqs, gbs: int, dp: int, mbs: int):
    """First gbs sequences + carryover (workload.py:265-278)."""
    if gbs % (dp * mbs) != 0:
        raise OracleConfigError(
            f"global batch {gbs} not divisible by dp {dp} x microbatch size {mbs}")
    if len(seqs) < gbs:
        raise ValueError(f"need {gbs} sequences, have {len(seqs)}")
    return seqs[:gbs], seqs[gbs:]


def generate(descs: dict, phases, linear: bool, step: int, seed: int, gbs: int,
             dp: int, mbs: int, capacity: int, carry=None):
    """One step of draw -> pack -> batch (workload.py:281-305).

    Returns (batch_seqs, carryover, samples_drawn, chunk_sizes).
    """
    seqs = list(carry or [])
    recipe = recipe_at(phases, step, linear)
    mean_len = np.mean([descs[nm]["mean"] for nm, r in recipe if r > 0])
    id_base = step * 1_000_000
    drawn, chunks = [], []
    draw = 0
    while len(seqs) < gbs:
        need = (gbs - len(seqs) + 1) * capacity
        n = max(int(need / mean_len) + 1, 16)
        chunk = draw_step(descs, phases, linear, step, n, seed + draw, id_base)
        id_base += n
        draw += 1
        drawn.extend(chunk)
        chunks.append(n)
        seqs.extend(ffd(chunk, capacity))
        if draw > 64:
            raise RuntimeError("packing failed to reach the global batch size")
    batch, rest = take_batch(seqs, gbs, dp, mbs)
    return batch, rest, drawn, chunks


def descs_from_config(cfg_datasets: dict, names) -> dict:
    """Descriptor dicts from paper_2605_08962_b200.configs.DATASETS rows."""
    out = {}
    for nm in names:
        modality, mean, max_len = cfg_datasets[nm]
        out[nm] = dict(name=nm, modality=modality, mean=mean, max_len=max_len)
    return out
