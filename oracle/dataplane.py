"""Fake-world data plane: every rank simulated in one process — TEST INFRASTRUCTURE ONLY.

There is no reference code for the data plane (the reference never moves
token data; pkg/src/muxsim/costs.py:84-105 models the
collectives as alpha-beta formulas).  Semantics follow SPEC.md:402 (data
all-to-all of grouped_reorder), SPEC.md:408-416 (restore_order)
(Ulysses reshard) and PAPER.md:1108-1114; the layout choices are the ones
recorded in oracle/planner.py.  Parity for this part is defined here, not
pinned by the reference ("parity unpinned" for the data plane).
"""

from __future__ import annotations

import numpy as np

M32 = np.uint32(0xFFFFFFFF)


def _mix32(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16)
    x = (x * np.uint32(0x85EBCA6B)).astype(np.uint32)
    x ^= x >> np.uint32(13)
    x = (x * np.uint32(0xC2B2AE35)).astype(np.uint32)
    x ^= x >> np.uint32(16)
    return x


def standin(sample_id: int, length: int, width: int) -> np.ndarray:
    """E(id, t, c) as uint16 bf16 bits [length, width] (csrc/segcopy.cu standin)."""
    sid = int(sample_id) & 0xFFFFFFFFFFFFFFFF
    lo = np.array([sid & 0xFFFFFFFF], np.uint32)
    hi = np.array([(sid >> 32) & 0xFFFFFFFF], np.uint32)
    sseed = _mix32(lo ^ _mix32((hi + np.uint32(0x632BE59B)).astype(np.uint32)))
    t = np.arange(length, dtype=np.uint32)
    rs = _mix32((sseed + (t * np.uint32(0x9E3779B9)).astype(np.uint32)).astype(np.uint32))
    c = (np.arange(width, dtype=np.uint32) * np.uint32(0x85EBCA77)).astype(np.uint32)
    h = _mix32(rs[:, None] ^ c[None, :])
    bits = ((h >> np.uint32(31)) << np.uint32(15)) | \
           ((np.uint32(126) + ((h >> np.uint32(7)) & np.uint32(1))) << np.uint32(7)) | \
           (h & np.uint32(0x7F))
    return bits.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16 bits (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    return ((u + rounding) >> np.uint32(16)).astype(np.uint16)


def run_world(plan: dict, table: dict, world: int, arenas, d_in, d_ret, d_llm,
              projector=None, encoder_out=None):
    """Move every row of one step through all ranks.

    arenas[r][g]: uint16 [arena_rows[r][g], d_in[g]] loader payload of rank r.
    projector: None (rows returned as-is, d_ret == d_llm) or per group
    (W bf16-bits [d_llm, d_enc], b bf16-bits [d_llm] or None) applied with
    fp32 accumulation and rounded to bf16.
    encoder_out: optional override of the encoder stand-in per (rank, group).
    Returns (recv[r][g], enc_out[r][g], llm[r]) as uint16 arrays.
    """
    ids = np.asarray(table["ids"])
    lens = np.asarray(table["lens"])
    G = len(d_in)
    recv = [[np.zeros((int(plan["recv_rows"][r, g]), d_in[g]), np.uint16) for g in range(G)]
            for r in range(world)]
    enc_out = [[np.zeros((int(plan["recv_rows"][r, g]), d_ret[g]), np.uint16) for g in range(G)]
               for r in range(world)]
    items = np.flatnonzero(plan["enc"] >= 0).tolist()
    for i in items:
        g, L = int(plan["group"][i]), int(lens[i])
        o, e = int(plan["origin"][i]), int(plan["enc"][i])
        a, b = int(plan["arena_off"][i]), int(plan["enc_off"][i])
        recv[e][g][b:b + L] = arenas[o][g][a:a + L]
        if encoder_out is None:
            enc_out[e][g][b:b + L] = standin(int(ids[i]), L, d_ret[g])
    if encoder_out is not None:
        enc_out = encoder_out
    llm = [np.zeros((int(plan["llm_rows"][r]), d_llm), np.uint16) for r in range(world)]
    for (i, src, dst_rank, dst_row, n) in plan["pieces"]:
        g, e = int(plan["group"][i]), int(plan["enc"][i])
        rows = enc_out[e][g][src:src + n]
        if projector is not None:
            W, bias = projector[g]
            x = bf16_bits_to_f32(rows)
            y = x @ bf16_bits_to_f32(W).T
            if bias is not None:
                y = y + bf16_bits_to_f32(bias)[None, :]
            rows = f32_to_bf16_bits(y.astype(np.float32))
        llm[dst_rank][dst_row:dst_row + n] = rows
    return recv, enc_out, llm


def pieces_by_rank(plan: dict, me: int):
    """Return pieces whose encoder rank is `me`, as (src_row, dst_row, rows,
    group, dst_rank) in table order — the GPU's return segment table."""
    out = []
    for (i, src, dst_rank, dst_row, n) in plan["pieces"]:
        if int(plan["enc"][i]) == me and n > 0:
            out.append((src, dst_row, n, int(plan["group"][i]), dst_rank))
    return np.array(out, np.int64).reshape(-1, 5)


def dispatch_by_rank(plan: dict, lens, me: int):
    """Dispatch segments of origin rank `me` in table order: (src_row, dst_row,
    rows, group, dst_rank) — the GPU's dispatch segment table."""
    out = []
    for i in np.flatnonzero(plan["enc"] >= 0).tolist():
        if int(plan["origin"][i]) == me and int(lens[i]) > 0:
            out.append((int(plan["arena_off"][i]), int(plan["enc_off"][i]), int(lens[i]),
                        int(plan["group"][i]), int(plan["enc"][i])))
    return np.array(out, np.int64).reshape(-1, 5)


def grad_by_rank(plan: dict, me: int):
    """Gradient-return segments of LLM rank `me` (the gradient path
    of restore_order): (src LLM row on me, dst encoder row, rows, group, encoder
    rank), in table order and, within a sample, in token order."""
    out = []
    for (i, src, dst_rank, dst_row, n) in plan["pieces"]:
        if dst_rank == me and n > 0:
            out.append((dst_row, src, n, int(plan["group"][i]), int(plan["enc"][i])))
    return np.array(out, np.int64).reshape(-1, 5)


def run_grad(plan: dict, world: int, dy, d_row):
    """dY rows of every LLM rank [llm_rows[r], d_row] -> each encoder rank's
    gradient buffer per group [recv_rows[e][g], d_row] in encoder order."""
    G = plan["recv_rows"].shape[1]
    grad = [[np.zeros((int(plan["recv_rows"][e, g]), d_row), dy[0].dtype) for g in range(G)]
            for e in range(world)]
    for (i, src, dst_rank, dst_row, n) in plan["pieces"]:
        g, e = int(plan["group"][i]), int(plan["enc"][i])
        grad[e][g][src:src + n] = dy[dst_rank][dst_row:dst_row + n]
    return grad


# ------------------------------------------------------------------ text rows
def text_offsets(table: dict) -> np.ndarray:
    """Offset of every text sample's token ids in the step's token array: the
    text samples of the step table (batch or not) in table order."""
    lens = np.asarray(table["lens"], np.int64)
    text = np.array([m == 0 for m in table["mods"]], bool)
    off = np.zeros(len(lens), np.int64)
    off[1:] = np.cumsum(np.where(text, lens, 0))[:-1]
    return np.where(text, off, -1)


def text_by_rank(plan: dict, table: dict, me: int):
    """Text segments of LLM rank `me`: (token offset, dst row, rows), table
    order then token order."""
    toff = text_offsets(table)
    out = [(int(toff[i]) + t0, drow, n) for (i, t0, dr, drow, n) in plan["text_pieces"]
           if dr == me]
    return np.array(out, np.int64).reshape(-1, 3)


def run_text(plan: dict, table: dict, world: int, tokens, emb, llm):
    """Write every rank's text rows: llm[r][row] = emb[tokens[offset + t]]."""
    toff = text_offsets(table)
    for (i, t0, dr, drow, n) in plan["text_pieces"]:
        ids = tokens[int(toff[i]) + t0:int(toff[i]) + t0 + n]
        llm[dr][drow:drow + n] = emb[ids]
    return llm
