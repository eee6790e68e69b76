"""Device planner: one step table in, one plan blob out (libmuxb200 K_ffd + K_finalize).

A *step table* lists the samples of one training step in table order: the
carried-over samples first (sequence/span order), then every drawn chunk in
draw order — exactly what ``generate_batch`` packs
(pkg/src/muxsim/workload.py:281-305).  The plan holds, bit-identically to
oracle/planner.py: FFD placement (workload.py:240-262), the global batch and
replica slice (:265-278, :177-180), Ulysses shard geometry,
origins, encoder assignment (LPT or KK), encoder order,
and the segment tables that drive the copy kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import PlanCfg, PlanLayout
from .configs import GROUP_OF_MOD
from .workload import MODALITY_CODE, PackedSequence, Sample

METHODS = {"lpt": _lib.LPT, "kk": _lib.KK, "lpt_local": _lib.LPT_LOCAL,
           "lpt_local_rw": _lib.LPT_LOCAL_RW}
DEFAULT_CHUNK_BYTES = 32768


def _stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


@dataclass
class StepTable:
    """Host (numpy) step table."""

    lens: np.ndarray       # int32[S]
    mods: np.ndarray       # int32[S] modality codes (text 0, image 1, video 2, audio 3)
    ids: np.ndarray        # int64[S]
    carry_seq: np.ndarray  # int32[n_carry]
    n_carry_seqs: int
    chunk_off: np.ndarray  # int32[n_chunks + 1], chunk_off[0] == n_carry

    @property
    def S(self) -> int:
        return int(self.lens.shape[0])

    @property
    def n_carry(self) -> int:
        return int(self.carry_seq.shape[0])

    @property
    def n_chunks(self) -> int:
        return int(self.chunk_off.shape[0]) - 1

    @staticmethod
    def from_chunks(carry: list[PackedSequence], chunks: list[list[Sample]],
                    modality_of: dict | None = None) -> "StepTable":
        """carry: PackedSequences carried in; chunks: drawn Sample lists;
        modality_of: sample id -> Modality for the carried samples."""
        lens, mods, ids, cseq = [], [], [], []
        for q, seq in enumerate(carry):
            for sid, tok in seq.spans:
                lens.append(tok)
                mods.append(MODALITY_CODE[modality_of[sid]])
                ids.append(sid)
                cseq.append(q)
        off = [len(lens)]
        for ch in chunks:
            for s in ch:
                lens.append(s.length)
                mods.append(MODALITY_CODE[s.modality])
                ids.append(s.id)
            off.append(len(lens))
        return StepTable(np.asarray(lens, np.int32), np.asarray(mods, np.int32),
                         np.asarray(ids, np.int64), np.asarray(cseq, np.int32), len(carry),
                         np.asarray(off, np.int32))

    def shard(self, rank: int, world: int) -> "StepTable":
        """The share of this step a decentralized loader on `rank` holds
        (PAPER.md:1104): carried sequences and drawn chunks split into `world`
        contiguous ranges in rank order (numpy array_split); carry sequence ids
        and chunk offsets are local.  gather_table reassembles the step."""
        qs = np.array_split(np.arange(self.n_carry_seqs), world)[rank]
        cs = np.array_split(np.arange(self.n_chunks), world)[rank]
        q0 = int(qs[0]) if len(qs) else 0
        carry = np.flatnonzero(np.isin(self.carry_seq, qs)) if len(qs) else np.zeros(0, np.int64)
        rows = [int(i) for i in carry]
        sizes = []
        for c in cs:
            lo, hi = int(self.chunk_off[c]), int(self.chunk_off[c + 1])
            rows += range(lo, hi)
            sizes.append(hi - lo)
        rows = np.asarray(rows, np.int64)
        off = np.concatenate([[len(carry)], len(carry) + np.cumsum(sizes, dtype=np.int64)])
        return StepTable(self.lens[rows].astype(np.int32), self.mods[rows].astype(np.int32),
                         self.ids[rows].astype(np.int64),
                         (self.carry_seq[carry] - q0).astype(np.int32), len(qs),
                         off.astype(np.int32))

    def record(self, cap_rows: int, cap_chunks: int) -> np.ndarray:
        """This shard as one metadata record (int32 words, include/mux_b200.h
        mux_assemble_table) for the all-gather."""
        S, nc, nch = self.S, self.n_carry, self.n_chunks
        if S > cap_rows or nch > cap_chunks:
            raise ValueError(f"shard of {S} rows / {nch} chunks exceeds the record capacity "
                             f"{cap_rows} / {cap_chunks}")
        rec = np.zeros(_lib.lib().mux_meta_record_words(cap_rows, cap_chunks), np.int32)
        rec[:4] = (nc, self.n_carry_seqs, S - nc, nch)
        rec[4:4 + 2 * cap_rows].view(np.int64)[:S] = self.ids
        o = 4 + 2 * cap_rows
        rec[o:o + S] = self.lens
        rec[o + cap_rows:o + cap_rows + S] = self.mods
        rec[o + 2 * cap_rows:o + 2 * cap_rows + nc] = self.carry_seq
        rec[o + 3 * cap_rows:o + 3 * cap_rows + nch] = np.diff(self.chunk_off)
        return rec

    def blob(self) -> np.ndarray:
        """One int64 array: ids | int32(lens, mods, carry_seq, chunk_off)."""
        S, nc, nch = self.S, self.n_carry, self.n_chunks
        n32 = 2 * S + nc + nch + 1
        out = np.zeros(S + (n32 + 1) // 2, np.int64)
        out[:S] = self.ids
        v = out[S:].view(np.int32)
        v[:S] = self.lens
        v[S:2 * S] = self.mods
        v[2 * S:2 * S + nc] = self.carry_seq
        v[2 * S + nc:2 * S + nc + nch + 1] = self.chunk_off
        return out


class DeviceTable:
    """A StepTable resident in device memory (one H2D copy)."""

    def __init__(self, table: StepTable, device, host_blob: torch.Tensor | None = None):
        """Copy `table` to `device`.  host_blob: the table's blob() already in
        pinned host memory (the copy is then asynchronous on the current stream)."""
        self.table = table
        if host_blob is None:
            self.blob = torch.from_numpy(table.blob()).to(device)
        else:
            self.blob = host_blob.to(device, non_blocking=True)
        S, nc = table.S, table.n_carry
        base = self.blob.data_ptr()
        self.ids = base
        i32 = base + 8 * S
        self.lens = i32
        self.mods = i32 + 4 * S
        self.carry_seq = i32 + 8 * S
        self.chunk_off = i32 + 4 * (2 * S + nc)

    @classmethod
    def from_blob(cls, table: StepTable, blob: torch.Tensor) -> "DeviceTable":
        """A view of a step-table blob already on the device (e.g. uploaded by a
        loader on its own stream): no copy."""
        return _device_table_from_blob(table, blob)


def _device_table_from_blob(table: StepTable, blob: torch.Tensor) -> "DeviceTable":
    dt = DeviceTable.__new__(DeviceTable)
    dt.table, dt.blob = table, blob
    S, nc = table.S, table.n_carry
    base = blob.data_ptr()
    dt.ids = base
    dt.lens, dt.mods = base + 8 * S, base + 12 * S
    dt.carry_seq, dt.chunk_off = base + 16 * S, base + 16 * S + 4 * nc
    return dt


class GatheredTable:
    """Step table assembled on the device from every rank's metadata record:
    the host holds only the sizes (what PlanCfg needs); the per-sample arrays
    are read back from the device blob on demand (e.g. plan.check's error
    message), never needed on the data path."""

    def __init__(self, blob: torch.Tensor, S: int, n_carry: int, n_carry_seqs: int,
                 n_chunks: int):
        self.dev_blob, self.S, self.n_carry = blob, S, n_carry
        self.n_carry_seqs, self.n_chunks = n_carry_seqs, n_chunks
        self._host = None

    def host(self) -> StepTable:
        if self._host is None:
            b = self.dev_blob.cpu().numpy()
            S, nc, nch = self.S, self.n_carry, self.n_chunks
            v = b[S:].view(np.int32)
            self._host = StepTable(v[:S].copy(), v[S:2 * S].copy(), b[:S].copy(),
                                   v[2 * S:2 * S + nc].copy(), self.n_carry_seqs,
                                   v[2 * S + nc:2 * S + nc + nch + 1].copy())
        return self._host

    ids = property(lambda self: self.host().ids)
    lens = property(lambda self: self.host().lens)
    mods = property(lambda self: self.host().mods)
    carry_seq = property(lambda self: self.host().carry_seq)
    chunk_off = property(lambda self: self.host().chunk_off)


def gather_table(shard: StepTable, device, group=None, cap_rows: int = 2048,
                 cap_chunks: int = 64, stream=None) -> "DeviceTable":
    """Decentralized metadata all-gather:
    this rank's loader share -> one record -> all_gather_into_tensor over the
    process group (NCCL over NVLink) -> mux_assemble_table on the device.  Only
    the 4-word record headers come back to the host (PlanCfg's sizes); run it
    on the planner's side stream one step ahead, as a loader prefetches."""
    import torch.distributed as dist
    L = _lib.lib()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    with torch.cuda.stream(s):
        rec = torch.from_numpy(shard.record(cap_rows, cap_chunks)).to(device, non_blocking=True)
        if world > 1:
            allrec = torch.empty(world * rec.numel(), dtype=torch.int32, device=device)
            dist.all_gather_into_tensor(allrec, rec, group=group)
        else:
            allrec = rec
        hdr = allrec.view(world, -1)[:, :4].cpu().numpy().astype(np.int64)
        nc, ncs, nk, nch = (int(x) for x in hdr.sum(0))
        S = nc + nk
        words = S + (2 * S + nc + nch + 1 + 1) // 2
        blob = torch.empty(max(words, 1), dtype=torch.int64, device=device)
        err = torch.zeros(1, dtype=torch.int32, device=device)
        _lib.check(L.mux_assemble_table(allrec.data_ptr(), world, cap_rows, cap_chunks,
                                        blob.data_ptr(), blob.numel(), err.data_ptr(),
                                        s.cuda_stream), "mux_assemble_table")
    table = GatheredTable(blob, S, nc, ncs, nch)
    return _device_table_from_blob(table, blob)


def make_cfg(table: StepTable, capacity: int, gbs: int = 0, dp: int = 1, sp: int = 1,
             world: int = 1, mbs: int = 1, method: str = "lpt", pooled: bool = False,
             me: int = 0, mode: int = _lib.MODE_STEP, row_bytes_in=(1176, 1024),
             row_bytes_ret=(8192, 8192), chunk_bytes: int = DEFAULT_CHUNK_BYTES,
             ret_mode: int = _lib.RET_FINAL, row_bytes_grad=None, lssp_sp: int = 0,
             lssp_eta: int = 0, reshard: str = "ulysses", cp_threshold: int = 0,
             text_embed: bool = False, reorder_group: int = 0, cost=None) -> PlanCfg:
    """One step's planner configuration (include/mux_b200.h mux_plan_cfg).
    lssp_sp > 0 turns on the LSSP eta split (samples longer than lssp_eta are
    encoded as token shards over groups of lssp_sp ranks; oracle/lssp.py).
    reshard: LLM placement over each replica's sp ranks, "ulysses" (uniform
    shards) or "cp_hybrid" (long samples split, short ones whole by LPT;
    oracle/cphybrid.py), cp_threshold 0 = capacity / sp.  reorder_group: ranks
    per reorder group (0 = the whole world).  cost: None (token
    counts) or per-encoder-group (lin, quad) with cost = lin L + quad L^2 —
    costs.flops_forward, see costs.encoder_cost_params."""
    if reshard not in _lib.RESHARD:
        raise ValueError(f"unknown reshard variant {reshard!r}")
    if method not in METHODS:
        raise ValueError(f"unknown balance method {method!r}")
    c = PlanCfg()
    c.S, c.n_carry, c.n_carry_seqs, c.n_chunks = table.S, table.n_carry, table.n_carry_seqs, \
        table.n_chunks
    c.capacity, c.gbs, c.dp, c.sp, c.world, c.mbs = capacity, gbs, dp, sp, world, mbs
    c.method, c.pooled, c.me, c.mode = METHODS[method], int(pooled), me, mode
    for g in range(_lib.N_GROUPS):
        c.row_bytes_in[g] = row_bytes_in[g]
        c.row_bytes_ret[g] = row_bytes_ret[g]
    c.chunk_bytes = chunk_bytes
    c.ret_mode = ret_mode
    for g in range(_lib.N_GROUPS):
        c.row_bytes_grad[g] = 0 if row_bytes_grad is None else row_bytes_grad[g]
    c.lssp_sp, c.lssp_eta = int(lssp_sp), int(lssp_eta)
    c.reshard, c.cp_threshold = _lib.RESHARD[reshard], int(cp_threshold)
    c.text_embed = int(bool(text_embed))
    c.reorder_group = int(reorder_group)
    if cost is None:
        c.cost_model = _lib.COST_TOKENS
    else:
        c.cost_model = _lib.COST_FLOPS
        for g in range(_lib.N_GROUPS):
            c.cost_lin[g], c.cost_quad[g] = float(cost[g][0]), float(cost[g][1])
    return c


def layout_of(cfg: PlanCfg) -> PlanLayout:
    L = PlanLayout()
    _lib.check(_lib.lib().mux_plan_layout_of(C.byref(cfg), C.byref(L)), "plan layout")
    return L


class Plan:
    """A device plan blob plus typed views of its arrays."""

    I32 = ("seq", "off", "span", "origin", "origin_pos", "group", "enc", "llm_rank",
           "bin_of", "fills", "nspans", "cu", "shard_len", "shard_start", "dseg_group",
           "dseg_dst_rank", "rseg_group", "rseg_dst_rank", "chunk_nbins", "gseg_group",
           "gseg_dst_rank", "lssp_state")
    I64 = ("arena_off", "enc_off", "llm_row", "row_base", "arena_rows", "recv_rows", "llm_rows",
           "lssp_row", "text_off", "tseg_src", "tseg_dst", "tseg_rows", "tseg_row0",
           "dseg_src_row", "dseg_dst_row", "dseg_rows", "rseg_src_row", "rseg_dst_row",
           "rseg_rows", "dseg_chunk0", "rseg_chunk0", "gseg_src_row", "gseg_dst_row",
           "gseg_rows", "gseg_chunk0")

    def __init__(self, cfg: PlanCfg, device, blob: torch.Tensor | None = None):
        self.cfg = cfg
        self.layout = layout_of(cfg)
        if blob is None or blob.numel() < self.layout.total:
            # zero-filled: the kernel's last-CTA ticket must start at 0
            blob = torch.zeros(self.layout.total, dtype=torch.uint8, device=device)
        self.blob = blob

    @property
    def ptr(self) -> int:
        return self.blob.data_ptr()

    def view(self, name: str, n: int) -> torch.Tensor:
        off = getattr(self.layout, name)
        dt = torch.int64 if name in self.I64 or name == "header" else torch.int32
        sz = 8 if dt == torch.int64 else 4
        return self.blob[off:off + sz * n].view(dt)

    def header(self) -> np.ndarray:
        return self.view("header", _lib.H_SLOTS).cpu().numpy()

    def check(self, table: StepTable) -> np.ndarray:
        """Synchronise, then raise the reference's exception for a failed plan."""
        h = np.ascontiguousarray(self.header())
        st = _lib.lib().mux_plan_check(C.byref(self.cfg), h.ctypes.data,
                                       np.ascontiguousarray(table.ids).ctypes.data,
                                       np.ascontiguousarray(table.lens).ctypes.data)
        _lib.check(st, "plan")
        return h

    def host(self) -> dict:
        """All per-sample / per-rank arrays on the host (tests and reporting)."""
        c, h = self.cfg, self.header()
        S, W, G = c.S, max(c.world, 1), _lib.N_GROUPS
        gb = max(c.gbs, 1) * max(c.sp, 1)
        out = {"header": h}
        for nm in ("seq", "off", "span", "origin", "origin_pos", "group", "enc", "arena_off",
                   "enc_off", "llm_rank", "llm_row"):
            out[nm] = self.view(nm, S).cpu().numpy()
        nseq = int(h[_lib.H_N_SEQ]) if h[_lib.H_N_SEQ] >= 0 else 0
        out["fills"] = self.view("fills", nseq).cpu().numpy()
        out["nspans"] = self.view("nspans", nseq).cpu().numpy()
        if c.mode == _lib.MODE_STEP and h[_lib.H_STATUS] == 0:
            out["cu"] = self.view("cu", c.gbs + 1).cpu().numpy()
            out["shard_len"] = self.view("shard_len", gb).cpu().numpy()
            out["shard_start"] = self.view("shard_start", gb).cpu().numpy()
            out["row_base"] = self.view("row_base", gb).cpu().numpy()
            out["arena_rows"] = self.view("arena_rows", W * G).cpu().numpy().reshape(W, G)
            out["recv_rows"] = self.view("recv_rows", W * G).cpu().numpy().reshape(W, G)
            out["llm_rows"] = self.view("llm_rows", W).cpu().numpy()
            nd, nr = int(h[_lib.H_N_DISPATCH]), int(h[_lib.H_N_RETURN])
            ng = int(h[_lib.H_N_GRAD])
            out["gseg"] = np.stack([self.view(k, ng).cpu().numpy().astype(np.int64) for k in (
                "gseg_src_row", "gseg_dst_row", "gseg_rows", "gseg_group", "gseg_dst_rank")],
                axis=1) if ng else np.zeros((0, 5), np.int64)
            out["dseg"] = np.stack([self.view("dseg_src_row", nd).cpu().numpy(),
                                    self.view("dseg_dst_row", nd).cpu().numpy(),
                                    self.view("dseg_rows", nd).cpu().numpy(),
                                    self.view("dseg_group", nd).cpu().numpy().astype(np.int64),
                                    self.view("dseg_dst_rank", nd).cpu().numpy().astype(np.int64)],
                                   axis=1) if nd else np.zeros((0, 5), np.int64)
            if c.text_embed:
                nt = int(h[_lib.H_N_TEXT])
                out["text_off"] = self.view("text_off", S).cpu().numpy()
                out["tseg"] = np.stack([self.view(k, nt).cpu().numpy() for k in (
                    "tseg_src", "tseg_dst", "tseg_rows")], axis=1) if nt else \
                    np.zeros((0, 3), np.int64)
            if c.lssp_sp > 0:
                out["lssp_state"] = self.view("lssp_state", S).cpu().numpy()
                out["lssp_row"] = self.view("lssp_row", S * _lib.LSSP_MAX).cpu().numpy() \
                    .reshape(S, _lib.LSSP_MAX)[:, :c.lssp_sp]
            out["rseg"] = np.stack([self.view("rseg_src_row", nr).cpu().numpy(),
                                    self.view("rseg_dst_row", nr).cpu().numpy(),
                                    self.view("rseg_rows", nr).cpu().numpy(),
                                    self.view("rseg_group", nr).cpu().numpy().astype(np.int64),
                                    self.view("rseg_dst_rank", nr).cpu().numpy().astype(np.int64)],
                                   axis=1) if nr else np.zeros((0, 5), np.int64)
        return out


def plan_step(dtab: DeviceTable, cfg: PlanCfg, plan: Plan | None = None, stream=None) -> Plan:
    """Launch the device planner (stream-ordered, no host sync)."""
    if plan is None or plan.blob.numel() < layout_of(cfg).total:
        old = plan
        # zero-fill on the launching stream (the ticket must read 0), with headroom
        # so a ring slot is not re-allocated every time the step grows
        with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
            need = layout_of(cfg).total
            blob = torch.zeros(need + need // 2 if old is not None else need,
                               dtype=torch.uint8, device=dtab.blob.device)
            plan = Plan(cfg, dtab.blob.device, blob)
        if old is not None:  # other streams may still read the old blob
            old.blob.record_stream(torch.cuda.current_stream())
    else:
        plan.cfg = cfg
        plan.layout = layout_of(cfg)
    st = _lib.lib().mux_plan_step(C.byref(cfg), dtab.lens, dtab.mods, dtab.ids, dtab.carry_seq,
                                  dtab.chunk_off, plan.ptr, plan.blob.numel(),
                                  _stream_ptr(stream))
    _lib.check(st, "mux_plan_step")
    plan.lens_ptr, plan.ids_ptr = dtab.lens, dtab.ids  # the table the plan was made from
    return plan


def _spans_from(seq, span, ids, lens, base, nbins, capacity):
    """PackedSequences of bins [base, base+nbins) from per-sample (seq, span)."""
    out = [PackedSequence(capacity=capacity) for _ in range(nbins)]
    order = np.lexsort((span, seq))
    for i in order.tolist():
        out[int(seq[i]) - base].spans.append((int(ids[i]), int(lens[i])))
    return out


def device_pack(chunks: list[list[Sample]], capacity: int, device=None):
    """hybrid_pack of each chunk on the GPU, one launch for all chunks.

    Returns one list of PackedSequences per chunk.  Raises PackingError with
    the reference's message for the first oversize sample in input order
    (workload.py:245-248).
    """
    device = device or torch.device("cuda", torch.cuda.current_device())
    table = StepTable.from_chunks([], chunks)
    cfg = make_cfg(table, capacity, mode=_lib.MODE_PACK)
    plan = plan_step(DeviceTable(table, device), cfg)
    h = plan.check(table)
    S = table.S
    seq = plan.view("seq", S).cpu().numpy()
    span = plan.view("span", S).cpu().numpy()
    nb = plan.view("chunk_nbins", table.n_chunks).cpu().numpy()
    res, base = [], 0
    for k in range(table.n_chunks):
        lo, hi = int(table.chunk_off[k]), int(table.chunk_off[k + 1])
        res.append(_spans_from(seq[lo:hi], span[lo:hi], table.ids[lo:hi], table.lens[lo:hi],
                               base, int(nb[k]), capacity))
        base += int(nb[k])
    assert base == int(h[_lib.H_N_SEQ])
    return res


def group_of_modality(code: int) -> int:
    return GROUP_OF_MOD[int(code)]
