"""LSSP eta split on the data path — TEST INFRASTRUCTURE ONLY (CPU restatement).

Long-short sequence parallelism (`lssp_schedule`; PAPER.md:
684-685, Fig. 6): per microbatch, samples of length <= eta are encoded in the
DP state (each rank encodes its own samples whole); longer samples are encoded
in the SP state, sharded over the rank's Ulysses group with an all-to-all
around the encoder.  The reference has only the SPEC (no code), so this
module pins the data layout; parity of the CUDA path against it is bit-exact.

Pinned choices:
* a sample is SP-state iff len > eta ("length <= eta form
  DP-state work"); zero-length samples are DP;
* encoder SP group of rank e: the sp_enc consecutive ranks
  [e - e % sp_enc, e - e % sp_enc + sp_enc); world % sp_enc == 0;
* the balancer's assignment is kept: an SP sample's "home" e (its rank from
  LPT/KK) only decides its group and its order;
* each encoder buffer (rank r, group g) holds the DP region first — DP
  samples of home r in encoder order (origin rank, table order) — then the SP
  region — my shard of every SP sample homed in my group, ordered by (home
  rank, encoder order);
* shard k of a sample of length L: n_k = L // sp_enc + (k < L % sp_enc)
  tokens starting at k * (L // sp_enc) + min(k, L % sp_enc) (the Ulysses
  split of SPEC.md:457, pinned in SURVEY.md §8.1-6);
* the SP all-to-all is fused into the dispatch: the origin pushes each shard
  straight to its member (one hop), and the return pushes each member's rows
  straight to their LLM position.

Every encoder row goes back to exactly one LLM row; the "fragments" below are
the intersections of the LLM pieces (oracle/planner.py plan_step) with the
encoder shards, in (table order, token order) — the order of the GPU's
return and gradient segment tables.
"""

from __future__ import annotations

import numpy as np

from .dataplane import standin


def shard(L: int, sp: int, k: int) -> tuple[int, int]:
    """(start, rows) of shard k of an L-token sample over sp ranks."""
    b, r = divmod(int(L), sp)
    return k * b + min(k, r), b + (1 if k < r else 0)


def layout(plan: dict, lens, world: int, eta: int, sp_enc: int) -> dict:
    """LSSP placement on top of a step plan.

    Returns state[S] (0 DP, 1 SP, -1 not encoded), row[S, sp_enc] (DP: row of the
    sample at its home in column 0; SP: row of shard k on member base+k),
    recv_rows[world, 2], and fragments (i, t0, n, src_rank, src_row, dst_rank,
    dst_row, group) in table order, then token order."""
    if sp_enc < 1 or world % sp_enc:
        raise ValueError(f"sp_enc {sp_enc} must divide world {world}")
    lens = np.asarray(lens, np.int64)
    enc, grp, eoff = plan["enc"], plan["group"], plan["enc_off"]
    S = len(lens)
    items = [i for i in range(S) if enc[i] >= 0]
    state = np.full(S, -1, np.int64)
    for i in items:
        state[i] = 1 if lens[i] > eta else 0
    row = np.full((S, sp_enc), -1, np.int64)
    dp_rows = np.zeros((world, 2), np.int64)
    for i in sorted(items, key=lambda i: (enc[i], eoff[i])):   # encoder order per home
        if state[i] == 0:
            row[i, 0] = dp_rows[enc[i], grp[i]]
            dp_rows[enc[i], grp[i]] += lens[i]
    recv = dp_rows.copy()
    for i in sorted([i for i in items if state[i] == 1], key=lambda i: (enc[i], eoff[i])):
        base = int(enc[i]) - int(enc[i]) % sp_enc
        for k in range(sp_enc):
            _, n = shard(lens[i], sp_enc, k)
            row[i, k] = recv[base + k, grp[i]]
            recv[base + k, grp[i]] += n
    frags = []
    by_sample: dict[int, list] = {}
    for (i, src, dst_rank, dst_row, n) in plan["pieces"]:
        by_sample.setdefault(i, []).append((src - int(eoff[i]), dst_rank, dst_row, n))
    for i in items:  # table order
        pcs = sorted(by_sample.get(i, []))
        g = int(grp[i])
        for (t0, dst_rank, dst_row, n) in pcs:
            if state[i] == 0:
                frags.append((i, t0, n, int(enc[i]), int(row[i, 0]) + t0, dst_rank, dst_row, g))
                continue
            base = int(enc[i]) - int(enc[i]) % sp_enc
            for k in range(sp_enc):
                s0, nk = shard(lens[i], sp_enc, k)
                a, b = max(t0, s0), min(t0 + n, s0 + nk)
                if a < b:
                    frags.append((i, a, b - a, base + k, int(row[i, k]) + a - s0,
                                  dst_rank, dst_row + a - t0, g))
    return dict(state=state, row=row, recv_rows=recv, dp_rows=dp_rows, fragments=frags,
                sp_enc=sp_enc, eta=eta)


def dispatch_by_rank(plan: dict, lay: dict, lens, me: int):
    """Dispatch segments of origin `me` in table order (shards in k order):
    (src arena row, dst row, rows, group, dst rank)."""
    out = []
    sp = lay["sp_enc"]
    for i in np.flatnonzero(plan["enc"] >= 0).tolist():
        L = int(lens[i])
        if int(plan["origin"][i]) != me or L == 0:
            continue
        g, e, a = int(plan["group"][i]), int(plan["enc"][i]), int(plan["arena_off"][i])
        if lay["state"][i] == 0:
            out.append((a, int(lay["row"][i, 0]), L, g, e))
            continue
        base = e - e % sp
        for k in range(sp):
            s0, n = shard(L, sp, k)
            if n:
                out.append((a + s0, int(lay["row"][i, k]), n, g, base + k))
    return np.array(out, np.int64).reshape(-1, 5)


def return_by_rank(lay: dict, me: int):
    """Return segments whose encoder rows live on `me`: (src row, dst row,
    rows, group, dst rank)."""
    out = [(f[4], f[6], f[2], f[7], f[5]) for f in lay["fragments"] if f[3] == me]
    return np.array(out, np.int64).reshape(-1, 5)


def grad_by_rank(lay: dict, me: int):
    """Gradient segments of LLM rank `me`: (src LLM row, dst encoder row, rows,
    group, encoder rank)."""
    out = [(f[6], f[4], f[2], f[7], f[3]) for f in lay["fragments"] if f[5] == me]
    return np.array(out, np.int64).reshape(-1, 5)


def run_world(plan: dict, lay: dict, table: dict, world: int, arenas, d_in, d_ret, d_llm):
    """All ranks of one LSSP step in one process: (recv, enc_out, llm) per rank,
    uint16 bf16 bits; the encoder stand-in is E(id, t, c) with t the token index
    within the whole sample, whichever rank computes it."""
    ids, lens = np.asarray(table["ids"]), np.asarray(table["lens"], np.int64)
    sp = lay["sp_enc"]
    recv = [[np.zeros((int(lay["recv_rows"][r, g]), d_in[g]), np.uint16) for g in range(2)]
            for r in range(world)]
    enc_out = [[np.zeros((int(lay["recv_rows"][r, g]), d_ret[g]), np.uint16) for g in range(2)]
               for r in range(world)]
    for i in np.flatnonzero(plan["enc"] >= 0).tolist():
        L, g, o, e = int(lens[i]), int(plan["group"][i]), int(plan["origin"][i]), int(plan["enc"][i])
        a = int(plan["arena_off"][i])
        if L == 0:
            continue
        full = standin(int(ids[i]), L, d_ret[g])
        if lay["state"][i] == 0:
            b = int(lay["row"][i, 0])
            recv[e][g][b:b + L] = arenas[o][g][a:a + L]
            enc_out[e][g][b:b + L] = full
            continue
        base = e - e % sp
        for k in range(sp):
            s0, n = shard(L, sp, k)
            b = int(lay["row"][i, k])
            recv[base + k][g][b:b + n] = arenas[o][g][a + s0:a + s0 + n]
            enc_out[base + k][g][b:b + n] = full[s0:s0 + n]
    llm = [np.zeros((int(plan["llm_rows"][r]), d_llm), np.uint16) for r in range(world)]
    for (i, t0, n, sr, srow, dr, drow, g) in lay["fragments"]:
        llm[dr][drow:drow + n] = enc_out[sr][g][srow:srow + n]
    return recv, enc_out, llm


def run_grad(lay: dict, world: int, dy, d_row):
    """dY rows of every LLM rank -> each encoder rank's gradient buffer in its
    LSSP encoder layout."""
    grad = [[np.zeros((int(lay["recv_rows"][e, g]), d_row), dy[0].dtype) for g in range(2)]
            for e in range(world)]
    for (i, t0, n, sr, srow, dr, drow, g) in lay["fragments"]:
        grad[sr][g][srow:srow + n] = dy[dr][drow:drow + n]
    return grad
