"""CPU restatement of the per-step planner — TEST INFRASTRUCTURE ONLY.

Inputs are a *step table*: the samples of one step in table order (carryover
samples first, in sequence/span order, then every drawn chunk in draw order),
exactly what workload.generate_batch (pkg/src/muxsim/workload.py:281-305)
consumes.  Output is the full plan as numpy arrays; the GPU planner must
reproduce every array bit-exactly.

Reference anchors:
  FFD per chunk ........ workload.py:240-262 (via oracle.workload.ffd)
  batch / replica slice  workload.py:265-278, :177-180
  LPT .................. BASELINE.json north_star ("greedy/LPT")
  kk_partition ......... SPEC.md:390-398 (pinned definition: SURVEY.md §8.1-1)
  grouped_reorder ...... SPEC.md:399-407 (pool window = whole step)
  restore_order ........ SPEC.md:408-416
  plan_reshard Ulysses . SPEC.md:453-470 (first F mod sp shards get +1)
Builder-defined layout (no reference code; "parity unpinned" by the
reference, defined here and in DESIGN.md §Layout):
  origin rank = LLM rank owning the sample's first token; loader arena of
  (rank, encoder group) in table order; encoder order (origin rank, table
  order); returned rows go straight to their LLM (rank, row).
"""

from __future__ import annotations

import numpy as np

from .workload import OracleConfigError, OraclePackingError

GROUP_OF_MOD = {0: -1, 1: 0, 2: 0, 3: 1}
N_GROUPS = 2


# ----------------------------------------------------------------------------
# assignment algorithms
# ----------------------------------------------------------------------------

def lpt_assign(costs, ids, g, init=None):
    """Longest-processing-time greedy: order by (-cost, id, index), each item to
    the least-loaded rank, lowest rank on ties.  Returns rank per item."""
    n = len(costs)
    order = sorted(range(n), key=lambda i: (-costs[i], ids[i], i))
    load = list(init) if init is not None else [0.0] * g
    out = [0] * n
    for i in order:
        r = min(range(g), key=lambda k: (load[k], k))
        out[i] = r
        load[r] = load[r] + costs[i]
    return out


def lpt_local_assign(costs, ids, origins, g, remote_weight=False):
    """Locality-first LPT (builder's variant of the north_star's greedy/LPT; the
    reference balances with KK over the whole group, moving
    almost every sample).  In LPT order (-cost, id, index): pass 1 keeps an item
    on its origin rank while that rank's kept load plus the item stays within
    T = sum(costs) / g; pass 2 places the remaining items by LPT (least load,
    lowest rank) on top of the kept loads.  Costs are integer token counts, so
    every sum is exact."""
    n = len(costs)
    order = sorted(range(n), key=lambda i: (-costs[i], ids[i], i))
    T = float(sum(costs)) / g
    kept = [0.0] * g
    out = [0] * n
    pool = []
    for i in order:
        o = origins[i]
        if kept[o] + costs[i] <= T:
            kept[o] = kept[o] + costs[i]
            out[i] = o
        else:
            pool.append(i)
    load = list(kept)
    for i in pool:
        # remote_weight: 9/8 of the cost on a rank other than the origin (exact:
        # integer costs, multiples of 1/8); the smallest resulting load wins
        ce = [costs[i] * 1.125 if remote_weight and k != origins[i] else costs[i]
              for k in range(g)]
        r = min(range(g), key=lambda k: (load[k] + ce[k], k))
        out[i] = r
        load[r] = load[r] + ce[r]
    return out


def kk_assign(weights, g):
    """g-way Karmarkar-Karp largest differencing.

    Pinned reading: every item starts as the g-tuple
    (w, 0, ..., 0); repeatedly pop the two tuples with the largest spread
    (max - min sum), ties to the lower minimum item index; the first popped
    is A.  Merge by pairing A's subsets sorted by (sum desc, min index asc)
    with B's sorted by (sum asc, min index asc).  The final subsets map to
    ranks 0..g-1 in (sum desc, min index asc) order.  g > n pads empty.
    """
    n = len(weights)
    if n == 0:
        return []
    inf = 1 << 62
    # a tuple = list of g subsets; subset = [sum, min_index, members]
    tuples = [[[weights[i], i, [i]]] + [[0.0 * weights[i], inf, []] for _ in range(g - 1)]
              for i in range(n)]

    def spread(t):
        sums = [s[0] for s in t]
        return max(sums) - min(sums)

    def tmin(t):
        return min(s[1] for s in t)

    alive = list(range(n))
    while len(alive) > 1:
        alive.sort(key=lambda k: (-spread(tuples[k]), tmin(tuples[k])))
        a, b = alive[0], alive[1]
        A = sorted(tuples[a], key=lambda s: (-s[0], s[1]))
        B = sorted(tuples[b], key=lambda s: (s[0], s[1]))
        merged = [[x[0] + y[0], min(x[1], y[1]), x[2] + y[2]] for x, y in zip(A, B)]
        tuples[a] = merged
        alive = [k for k in alive if k != b]
    final = sorted(tuples[alive[0]], key=lambda s: (-s[0], s[1]))
    out = [0] * n
    for rank, sub in enumerate(final):
        for i in sub[2]:
            out[i] = rank
    return out


def ulysses_split(fill, sp):
    """Shard lengths of a sequence of `fill` tokens over sp ranks; the first
    fill % sp shards get one extra token."""
    q, r = divmod(int(fill), sp)
    return [q + (1 if k < r else 0) for k in range(sp)]


# ----------------------------------------------------------------------------
# step plan
# ----------------------------------------------------------------------------

def plan_step(table, capacity, gbs, dp, sp, world, mbs=1, method="lpt", pooled=False,
              packed=None, reorder_group=0, cost=None):
    """Plan one step.  `table` dict: lens, mods, ids (arrays over S samples),
    carry_seq (array over the first n_carry samples: their carry sequence),
    n_carry_seqs, chunk_off (offsets of drawn chunks, first = n_carry).
    packed: optional (seq, off, span, fills) of an FFD placement computed
    elsewhere — bench.py's reference arm passes the reference's own
    hybrid_pack output (packed_from_sequences) and times only the rest here.
    reorder_group: ranks per reorder group (0 = world): a sample is
    balanced over the ranks of its origin's group only.  cost: None (token
    counts) or per-encoder-group (lin, quad) pairs, cost =
    lin * L + quad * L * L — costs.flops_forward (costs.py:108-124) with
    lin = 2 P, quad = 2 layers hidden, mult 1."""
    lens = np.asarray(table["lens"], dtype=np.int64)
    mods = np.asarray(table["mods"], dtype=np.int64)
    ids = np.asarray(table["ids"], dtype=np.int64)
    carry_seq = np.asarray(table.get("carry_seq", []), dtype=np.int64)
    n_carry_seqs = int(table.get("n_carry_seqs", 0))
    chunk_off = list(table["chunk_off"])
    S = len(lens)
    nc = len(carry_seq)
    if dp * sp != world:
        raise OracleConfigError(f"llm dp {dp} x sp {sp} != world {world}")

    # oversize: first offender in table order among drawn samples (workload.py:245)
    for i in range(nc, S):
        if lens[i] > capacity:
            raise OraclePackingError(
                f"sample {ids[i]} ({lens[i]} tokens) exceeds capacity {capacity}")

    if packed is not None:
        seq, off, span, fills = (np.asarray(a, np.int64) for a in packed)
        fills = fills.tolist()
        n_seq = len(fills)
    else:
        seq, off, span, fills, n_seq = _ffd_table(lens, ids, carry_seq, n_carry_seqs, chunk_off,
                                                  capacity)
    return _plan_packed(lens, mods, ids, seq, off, span, fills, n_seq, capacity, gbs, dp, sp,
                        world, mbs, method, pooled, reorder_group, cost)


def _ffd_table(lens, ids, carry_seq, n_carry_seqs, chunk_off, capacity):
    """Carry spans, then FFD of every drawn chunk (workload.py:240-262, :288)."""
    S, nc = len(lens), len(carry_seq)
    seq = np.full(S, -1, np.int64)
    off = np.zeros(S, np.int64)
    span = np.zeros(S, np.int64)
    fills = [0] * n_carry_seqs
    nspan = [0] * n_carry_seqs
    for i in range(nc):
        q = int(carry_seq[i])
        seq[i], off[i], span[i] = q, fills[q], nspan[q]
        fills[q] += int(lens[i])
        nspan[q] += 1
    base = n_carry_seqs
    for c in range(len(chunk_off) - 1):
        lo, hi = chunk_off[c], chunk_off[c + 1]
        idx = sorted(range(lo, hi), key=lambda i: (-lens[i], ids[i], i))
        bf = []
        for i in idx:
            for b, f in enumerate(bf):
                if f + lens[i] <= capacity:
                    break
            else:
                b = len(bf)
                bf.append(0)
                fills.append(0)
                nspan.append(0)
            q = base + b
            seq[i], off[i], span[i] = q, bf[b], nspan[q]
            bf[b] += int(lens[i])
            fills[q] = bf[b]
            nspan[q] += 1
        base += len(bf)
    return seq, off, span, fills, base


def packed_from_sequences(table, sequences):
    """(seq, off, span, fills) of a list of PackedSequences (carry first, then
    every chunk's hybrid_pack output in order) over the step table's rows.
    Sample ids are unique within a step (workload.py:225-236 id_base)."""
    ids = np.asarray(table["ids"], dtype=np.int64)
    row = {int(sid): i for i, sid in enumerate(ids.tolist())}
    S = len(ids)
    seq = np.full(S, -1, np.int64)
    off = np.zeros(S, np.int64)
    span = np.zeros(S, np.int64)
    fills = []
    for q, ps in enumerate(sequences):
        f = 0
        for k, (sid, tok) in enumerate(ps.spans):
            i = row[int(sid)]
            seq[i], off[i], span[i] = q, f, k
            f += int(tok)
        fills.append(f)
    return seq, off, span, fills


def sample_cost(L, group, cost):
    """Balancing cost of one sample (exact in fp64 for integer parameters)."""
    if cost is None:
        return float(L)
    lin, quad = cost[group]
    return float(lin) * float(L) + float(quad) * float(L) * float(L)


def _plan_packed(lens, mods, ids, seq, off, span, fills, n_seq, capacity, gbs, dp, sp, world,
                 mbs, method, pooled, reorder_group=0, cost=None):
    S = len(lens)
    if gbs % (dp * mbs) != 0:
        raise OracleConfigError(
            f"global batch {gbs} not divisible by dp {dp} x microbatch size {mbs}")
    if n_seq < gbs:
        raise ValueError(f"need {gbs} sequences, have {n_seq}")

    P = gbs // dp
    fills = np.asarray(fills, dtype=np.int64)
    in_batch = seq < gbs
    cu = np.zeros(gbs + 1, np.int64)
    cu[1:] = np.cumsum(fills[:gbs])

    # Ulysses shard geometry per batch sequence
    shard_len = np.array([ulysses_split(fills[q], sp) for q in range(gbs)],
                         dtype=np.int64).reshape(gbs, sp)
    shard_start = np.zeros((gbs, sp), np.int64)
    shard_start[:, 1:] = np.cumsum(shard_len[:, :-1], axis=1)
    # local row base of sequence q on its replica's shard-k rank
    row_base = np.zeros((gbs, sp), np.int64)
    llm_rows = np.zeros(world, np.int64)
    for q in range(gbs):
        r = q // P
        for k in range(sp):
            row_base[q, k] = llm_rows[r * sp + k]
            llm_rows[r * sp + k] += shard_len[q, k]

    def owner(q, pos):
        k = int(np.searchsorted(shard_start[q], pos, side="right") - 1)
        return (q // P) * sp + k, k

    group = np.array([GROUP_OF_MOD[int(m)] for m in mods], dtype=np.int64) if S else \
        np.zeros(0, np.int64)
    origin = np.full(S, -1, np.int64)
    origin_pos = np.full(S, -1, np.int64)
    for i in range(S):
        if in_batch[i]:
            q = int(seq[i])
            pos = min(int(off[i]), max(int(fills[q]) - 1, 0))
            origin[i] = owner(q, pos)[0]
    # origin_pos: (seq, span) order within each origin rank
    cnt = np.zeros(world, np.int64)
    for i in sorted(np.flatnonzero(in_batch).tolist(), key=lambda i: (seq[i], span[i])):
        origin_pos[i] = cnt[origin[i]]
        cnt[origin[i]] += 1

    enc_item = [i for i in range(S) if in_batch[i] and group[i] >= 0]
    arena_off = np.full(S, -1, np.int64)
    arena_rows = np.zeros((world, N_GROUPS), np.int64)
    for i in enc_item:   # table order
        arena_off[i] = arena_rows[origin[i], group[i]]
        arena_rows[origin[i], group[i]] += lens[i]

    enc = np.full(S, -1, np.int64)
    RG = reorder_group or world
    if world % RG:
        raise ValueError(f"reorder group {RG} must divide world {world}")
    pools = []  # (reorder group, encoder group or pooled), table order inside
    for rg in range(world // RG):
        mine = [i for i in enc_item if origin[i] // RG == rg]
        pools += [(rg, mine)] if pooled else [(rg, [i for i in mine if group[i] == q])
                                              for q in range(N_GROUPS)]
    for rg, items in pools:
        if not items:
            continue
        costs = [sample_cost(lens[i], group[i], cost) for i in items]
        if RG == 1:
            ranks = [0] * len(items)
        elif method == "lpt":
            ranks = lpt_assign(costs, [int(ids[i]) for i in items], RG)
        elif method == "kk":
            ranks = kk_assign(costs, RG)
        elif method in ("lpt_local", "lpt_local_rw"):
            ranks = lpt_local_assign(costs, [int(ids[i]) for i in items],
                                     [int(origin[i]) - rg * RG for i in items], RG,
                                     remote_weight=method == "lpt_local_rw")
        else:
            raise ValueError(f"unknown method {method!r}")
        for i, r in zip(items, ranks):
            enc[i] = rg * RG + r

    enc_off = np.full(S, -1, np.int64)
    recv_rows = np.zeros((world, N_GROUPS), np.int64)
    for i in sorted(enc_item, key=lambda i: (origin[i], i)):
        enc_off[i] = recv_rows[enc[i], group[i]]
        recv_rows[enc[i], group[i]] += lens[i]

    # return pieces: (sample, src row in encoder buffer, dst rank, dst row, rows)
    pieces = []
    for i in enc_item:
        q, r0, L = int(seq[i]), int(off[i]), int(lens[i])
        t = 0
        while t < L:
            pos = r0 + t
            rank, k = owner(q, pos)
            n = min(L - t, int(shard_start[q, k] + shard_len[q, k]) - pos)
            pieces.append((i, int(enc_off[i]) + t, rank,
                           int(row_base[q, k]) + pos - int(shard_start[q, k]), n))
            t += n
    # text samples' LLM pieces (token offset in the sample, dst rank, dst row, rows):
    # their rows come from the embedding table, not from an encoder
    text_pieces = []
    for i in range(S):
        if not in_batch[i] or group[i] >= 0:
            continue
        q, r0, L = int(seq[i]), int(off[i]), int(lens[i])
        t = 0
        while t < L:
            pos = r0 + t
            rank, k = owner(q, pos)
            n = min(L - t, int(shard_start[q, k] + shard_len[q, k]) - pos)
            text_pieces.append((i, t, rank, int(row_base[q, k]) + pos - int(shard_start[q, k]), n))
            t += n
    return dict(seq=seq, off=off, span=span, n_seq=n_seq, fills=fills, cu=cu,
                in_batch=in_batch, origin=origin, origin_pos=origin_pos, group=group,
                arena_off=arena_off, arena_rows=arena_rows, enc=enc, enc_off=enc_off,
                recv_rows=recv_rows, llm_rows=llm_rows, shard_len=shard_len,
                row_base=row_base, pieces=pieces, text_pieces=text_pieces, P=P)


def restore_order(plan):
    """Inverse of the reorder: for every encoder-side row
    block, where the origin rank keeps it.  Returns {(enc, group, enc_off):
    (origin, arena_off)}; exactness is checked by composition in the tests."""
    out = {}
    for i in np.flatnonzero(plan["enc"] >= 0).tolist():
        out[(int(plan["enc"][i]), int(plan["group"][i]), int(plan["enc_off"][i]))] = \
            (int(plan["origin"][i]), int(plan["arena_off"][i]))
    return out


def step_table(carry_seqs, drawn, chunk_sizes, modality_of):
    """Build a step table from generate_batch-shaped data.  carry_seqs: list of
    span lists; drawn: list of (id, modality, dataset, length); modality_of:
    id -> modality string for carry samples."""
    code = {"text": 0, "image": 1, "video": 2, "audio": 3}
    lens, mods, ids, carry_seq = [], [], [], []
    for q, spans in enumerate(carry_seqs):
        for sid, L in spans:
            lens.append(L)
            mods.append(code[modality_of[sid]])
            ids.append(sid)
            carry_seq.append(q)
    nc = len(lens)
    for sid, m, _, L in drawn:
        lens.append(L)
        mods.append(code[m])
        ids.append(sid)
    chunk_off = [nc]
    for n in chunk_sizes:
        chunk_off.append(chunk_off[-1] + n)
    return dict(lens=np.array(lens, np.int64), mods=np.array(mods, np.int64),
                ids=np.array(ids, np.int64), carry_seq=np.array(carry_seq, np.int64),
                n_carry_seqs=len(carry_seqs), chunk_off=chunk_off)


def plan_reshard(sequences, n_ranks, variant, cp_threshold=None, capacity=None):
    """Encoder -> LLM shard map, one sequence at a time.

    sequences: list of span lists [(sample id, tokens)].
    UlyssesUniform: each sequence's fill F splits into n_ranks contiguous
      shards, the first F mod n_ranks one token longer (pinned in
      SURVEY.md §8.1-6); a sample maps to every shard its token range touches.
    CpHybrid: samples longer than cp_threshold (default capacity / n_ranks,
      SPEC.md:497) split into n_ranks near-equal pieces (same rule), one per
      rank; shorter samples go whole to a rank by LPT whose initial loads are
      the long-sample pieces already on each rank.
    Returns {sample id: [(rank, start, end)]} (token ranges within the sample)
    and per-rank token counts per sequence.
    """
    smap, loads = {}, []
    for spans in sequences:
        if variant == "ulysses":
            F = sum(t for _, t in spans)
            lens = ulysses_split(F, n_ranks)
            starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
            pos = 0
            for sid, t in spans:
                pieces = []
                for k in range(n_ranks):
                    a, b = max(pos, int(starts[k])), min(pos + t, int(starts[k]) + lens[k])
                    if a < b:
                        pieces.append((k, a - pos, b - pos))
                smap[sid] = pieces
                pos += t
            loads.append(list(lens))
        elif variant == "cp_hybrid":
            thr = cp_threshold if cp_threshold is not None else capacity // n_ranks
            load = [0] * n_ranks
            short = []
            for idx, (sid, t) in enumerate(spans):
                if t > thr:
                    parts = ulysses_split(t, n_ranks)
                    off = 0
                    smap[sid] = []
                    for k, n in enumerate(parts):
                        smap[sid].append((k, off, off + n))
                        load[k] += n
                        off += n
                else:
                    short.append((idx, sid, t))
            if short:
                ranks = lpt_assign([float(t) for _, _, t in short], [sid for _, sid, _ in short],
                                   n_ranks, init=[float(x) for x in load])
                for (idx, sid, t), r in zip(short, ranks):
                    smap[sid] = [(r, 0, t)]
                    load[r] += t
            loads.append(load)
        else:
            raise ValueError(f"unknown reshard variant {variant!r}")
    return smap, loads


def assemble_records(records, cap_rows, cap_chunks):
    """Global step table from every rank's metadata record (rank order) — the
    CPU restatement of mux_assemble_table (csrc/meta.cu) for the decentralized
    metadata all-gather.  Builder-defined record layout:
    [n_carry_rows, n_carry_seqs, n_chunk_rows, n_chunks], ids int64[cap],
    lens, mods, local carry seq int32[cap], chunk sizes int32[cap_chunks]."""
    lens, mods, ids, cseq = [], [], [], []
    klens, kmods, kids, sizes = [], [], [], []
    q0 = 0
    for rec in records:
        rec = np.asarray(rec, np.int32)
        ncr, ncs, nkr, nk = (int(x) for x in rec[:4])
        rid = rec[4:4 + 2 * cap_rows].view(np.int64)
        o = 4 + 2 * cap_rows
        rl, rm = rec[o:o + cap_rows], rec[o + cap_rows:o + 2 * cap_rows]
        rc, rs = rec[o + 2 * cap_rows:o + 3 * cap_rows], rec[o + 3 * cap_rows:]
        ids += rid[:ncr].tolist(); lens += rl[:ncr].tolist(); mods += rm[:ncr].tolist()
        cseq += (rc[:ncr] + q0).tolist()
        kids += rid[ncr:ncr + nkr].tolist(); klens += rl[ncr:ncr + nkr].tolist()
        kmods += rm[ncr:ncr + nkr].tolist(); sizes += rs[:nk].tolist()
        q0 += ncs
    nc = len(ids)
    chunk_off = [nc]
    for n in sizes:
        chunk_off.append(chunk_off[-1] + n)
    return dict(lens=np.array(lens + klens, np.int64), mods=np.array(mods + kmods, np.int64),
                ids=np.array(ids + kids, np.int64), carry_seq=np.array(cseq, np.int64),
                n_carry_seqs=q0, chunk_off=chunk_off)
