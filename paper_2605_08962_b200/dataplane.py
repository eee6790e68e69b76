"""The per-step encoder<->LLM data path on B200: plan -> pack+dispatch -> return+scatter.

One process per GPU.  Every rank plans the whole step on its own GPU (the
plan is integer-only and bit-identical on every rank), then *pushes* its rows:

  pack + dispatch   loader arena rows -> the encoder rank's receive window,
                    written directly over NVLink (SPEC.md:402 data all-to-all;
                    PAPER.md:1108-1110 grouped reordering)
  return + scatter  encoder output rows -> their LLM rank's packed input at the
                    placeholder positions (SPEC.md:408-416 restore_order and
                    SPEC.md:462-470 plan_reshard, one hop instead of the
                    paper's send-then-reshard)
  projector         with a projector, the tcgen05 GEMM whose epilogue stores each
                    output row at its (rank, row); across GPUs see `MuxPath`.

Receive windows, LLM buffers and completion flags are torch symmetric-memory
allocations (CUDA VMM + IPC under the hood); the kernels get raw peer pointers.
There is no NCCL on the data path: no counts are exchanged, because every rank
already knows every offset.  At world 1 the same kernels run on local pointers.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _lib
from .planner import DeviceTable, Plan, StepTable, layout_of, make_cfg, plan_step, _stream_ptr

N_GROUPS = _lib.N_GROUPS


class _Window:
    """A buffer every rank can address: local tensor + per-rank pointers."""

    def __init__(self, nbytes: int, device, group=None, world: int = 1):
        nbytes = max(int(nbytes), 256)
        if world == 1:
            self.tensor = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self.ptrs = [self.tensor.data_ptr()]
            self.handle = None
        else:
            import torch.distributed._symmetric_memory as symm
            self.tensor = symm.empty(nbytes, dtype=torch.uint8, device=device)
            self.handle = symm.rendezvous(self.tensor, group)
            me = self.handle.rank
            delta = self.tensor.data_ptr() - self.handle.buffer_ptrs[me]
            self.ptrs = [p + delta for p in self.handle.buffer_ptrs]


def _ptr_table(ptrs, device) -> torch.Tensor:
    return torch.tensor([int(p) for p in ptrs], dtype=torch.int64, device=device)


def _event(timing: bool = False) -> torch.cuda.Event:
    return torch.cuda.Event(enable_timing=timing)


class MuxPath:
    """Per-rank data path for one workload shape.

    capacity/gbs/dp/sp/world follow the reference's GlobalBatch
    (workload.py:166-183) and the LLM layout of plan_reshard.
    d_in[g] is the loader row width of encoder group g (0 vision, 1 audio),
    d_enc[g] the encoder hidden, d_llm the LLM hidden.  projector=False
    returns d_llm-wide encoder rows bit-exactly; projector=True returns
    Y = X W_g^T (+ b_g) from d_enc-wide rows.

    Projector across GPUs (projector_return, env MUX_PROJECTOR_RETURN):
      "fused" (default)  the GEMM runs on the encoder rank (where LPT balanced
          the rows) and its epilogue stores every output row straight into the
          owner's packed buffer over NVLink: compute and collective in one kernel;
      "staged"  the narrow d_enc rows are pushed to the LLM owner's
          staging window (3.2x fewer NVLink bytes than d_llm rows) and the
          owner projects them on a projector stream, overlapped with the next
          step's dispatch and return (staging and LLM buffers alternate, so
          step k's LLM rows are final once the event `return_scatter` returns
          has fired and stay valid until step k+2's projector runs); the
          owners' rows are not balanced by the encoder-side LPT, so at 2 GPUs it
          measured no faster than "fused".

    Other options:
      method            encoder balancing: "lpt_local" (bench default), "lpt",
                        "kk", "lpt_local_rw";
      lssp_eta/lssp_sp  LSSP eta split: longer samples are encoded as token
                        shards over groups of lssp_sp ranks (None: off);
      reshard           LLM placement over each replica's sp ranks: "ulysses"
                        or "cp_hybrid" (cp_threshold, 0 = capacity / sp);
      text_embed        also emit text segments for `embed_text`;
      overlap_dispatch  `run_pipeline` dispatches step k+1 under step k's
                        return (E/D/R flag channels, alternating LLM buffers);
      reorder_group     balance each sample only over the ranks of its origin's
                        group of consecutive ranks (0 = world);
      cost              None (token counts) or per-group (lin, quad) flops
                        weights (costs.encoder_cost_params).
    """

    def __init__(self, *, capacity: int, gbs: int, dp: int, sp: int = 1, world: int = 1,
                 rank: int = 0, method: str = "lpt", pooled: bool = False,
                 d_in=(588, 512), d_enc=(1280, 1280), d_llm: int = 4096,
                 projector: bool = False, device=None, group=None, max_rows: int | None = None,
                 wait_timeout_ms: int = 20000, projector_return: str | None = None,
                 lssp_eta: int | None = None, lssp_sp: int = 1, reshard: str = "ulysses",
                 cp_threshold: int = 0, text_embed: bool = False,
                 overlap_dispatch: bool = False, reorder_group: int = 0, cost=None):
        self.capacity, self.gbs, self.dp, self.sp = capacity, gbs, dp, sp
        # balancing scope and cost (planner.make_cfg): reorder groups of
        # consecutive ranks (0 = world) and token or flops costs
        self.reorder_group, self.cost = reorder_group, cost
        self.world, self.rank, self.method, self.pooled = world, rank, method, pooled
        self.d_in, self.d_enc, self.d_llm = tuple(d_in), tuple(d_enc), d_llm
        self.projector = projector
        self.device = dev = device or torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.timeout_ms = wait_timeout_ms
        self.d_ret = tuple(d_enc) if projector else (d_llm, d_llm)
        mode = projector_return or os.environ.get("MUX_PROJECTOR_RETURN", "fused")
        if mode not in ("fused", "staged"):
            raise ValueError(f"projector_return must be 'fused' or 'staged', not {mode!r}")
        self.projector_return = mode
        # LSSP eta split: samples longer than lssp_eta are encoded
        # as token shards over groups of lssp_sp consecutive ranks (None: off)
        if lssp_eta is not None and (lssp_sp < 1 or world % lssp_sp):
            raise ValueError(f"lssp_sp {lssp_sp} must divide world {world}")
        self.lssp_eta, self.lssp_sp = lssp_eta, lssp_sp
        # LLM-side placement over each replica's sp ranks (reshard.plan_reshard)
        self.reshard, self.cp_threshold = reshard, cp_threshold
        # text tokens' embedding rows gathered into the same packed LLM buffer
        self.text_embed = text_embed
        self.staged = bool(projector and world > 1 and mode == "staged")
        self.ret_mode = _lib.RET_STAGED if self.staged else _lib.RET_FINAL
        rows = max_rows or gbs * capacity                       # all batch tokens
        llm_rows = (gbs // dp) * capacity // sp + gbs // dp + 1  # one rank's shards
        if reshard == "cp_hybrid":  # LPT may stack short samples on one CP rank
            llm_rows = (gbs // dp) * capacity
        self.max_rows, self.max_llm_rows = rows, llm_rows
        self.num_sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.gemm_ctas = 0  # 0: one CTA per SM; plan_ahead() leaves one SM to the planner

        # overlap_dispatch: step k+1's dispatch may run under step k's return (see
        # dispatch_overlapped); across GPUs the LLM buffers then alternate per step
        self.overlap_dispatch = overlap_dispatch
        self.recv = [_Window(rows * d_in[g] * 2, dev, group, world) for g in range(N_GROUPS)]
        n_llm = 2 if self.staged or (overlap_dispatch and world > 1) else 1
        self._nret = 0
        self.llm_bufs = [_Window(llm_rows * d_llm * 2, dev, group, world) for _ in range(n_llm)]
        # completion-flag channels (each its own epoch counter): R = return and
        # gradient exchanges, D = dispatch, E = "receive windows consumed"
        self.flags = _Window(8 * world, dev, group, world)
        self.flags.tensor.zero_()
        self.flags_d = _Window(8 * world, dev, group, world)
        self.flags_d.tensor.zero_()
        self.flags_e = _Window(8 * world, dev, group, world)
        self.flags_e.tensor.zero_()
        self.epoch_d = torch.zeros(1, dtype=torch.int64, device=dev)
        self.epoch_e = torch.zeros(1, dtype=torch.int64, device=dev)
        self._e_sent = 0  # E signals issued (host count = the device epoch_e)
        self._fuse_e = False  # the next fused projector launch carries the E signal
        self.enc_out = [torch.empty(rows * self.d_ret[g], dtype=torch.bfloat16, device=dev)
                        for g in range(N_GROUPS)]
        # copy counters x3 tables, then the projector's completion ticket
        self.sync = torch.zeros(8, dtype=torch.int32, device=dev)
        self.kernel_events = None  # (start, end) CUDA events around the return kernel
        # copy work unit and grid of the segment copies (tuning knobs; 0 = default grid)
        self.chunk_bytes = int(os.environ.get("MUX_CHUNK_BYTES", "32768"))
        self.copy_grid = int(os.environ.get("MUX_COPY_GRID", "0"))
        # an overlapped dispatch runs as lean copy CTAs (no shared memory) beside the
        # return: 2 per SM next to the projector GEMM (its registers and shared
        # memory leave room for no more), 3 per SM next to a return copy (a copy CTA
        # holds 16K registers: 4 per SM would leave none for the return kernel,
        # which then waits for the dispatch to drain)
        env_dg = os.environ.get("MUX_DISPATCH_GRID")
        if env_dg is not None:
            self.dispatch_grid = int(env_dg)
        elif overlap_dispatch:
            self.dispatch_grid = -(2 if projector else 3) * self.num_sms
        else:
            self.dispatch_grid = self.copy_grid
        self.epoch_ctr = torch.zeros(1, dtype=torch.int64, device=dev)
        # status word of the exchanges (the poison of segcopy.cu): a flag wait
        # that times out sets 1, one that sees a poisoned peer sets 2; later
        # copies and GEMMs then move nothing and pass the poison on, later waits
        # return at once.  run_pipeline mirrors it to the host asynchronously and
        # raises at its next call once the copy has landed; check_wait() syncs.
        self.wait_err = torch.zeros(1, dtype=torch.int32, device=dev)
        self._status_host = torch.zeros(1, dtype=torch.int32).pin_memory() if world > 1 else None
        self._status_ev = None
        self.step_done = None  # run_pipeline: the current step's "inputs no longer read" event
        self.recv_dst = _ptr_table([self.recv[g].ptrs[r] for r in range(world)
                                    for g in range(N_GROUPS)], dev)
        self.llm_dst = [_ptr_table(b.ptrs, dev) for b in self.llm_bufs]
        self.enc_src = _ptr_table([t.data_ptr() for t in self.enc_out], dev)
        self.flag_ptrs = _ptr_table(self.flags.ptrs, dev)
        self.flag_ptrs_d = _ptr_table(self.flags_d.ptrs, dev)
        self.flag_ptrs_e = _ptr_table(self.flags_e.ptrs, dev)
        self._arena_tables: dict = {}
        self._plan: Plan | None = None
        self._ring = None
        self.last_llm = 0
        if self.staged:
            self.stage = [[_Window(llm_rows * d_enc[g] * 2, dev, group, world)
                           for g in range(N_GROUPS)] for _ in range(2)]
            self.stage_dst = [_ptr_table([self.stage[b][g].ptrs[r] for r in range(world)
                                          for g in range(N_GROUPS)], dev) for b in range(2)]
            self._proj = torch.cuda.Stream(dev)
            self._ev_p = [None, None]
            self._kret = 0
            self.row_dst_b = [torch.empty(llm_rows, dtype=torch.int64, device=dev)
                              for _ in range(2)]
        if world > 1:
            torch.cuda.synchronize()
            self.flags.handle.barrier()
        if projector:
            self.weight = [None] * N_GROUPS
            self.bias = [None] * N_GROUPS
            self.row_dst = torch.empty(N_GROUPS * rows, dtype=torch.int64, device=dev)
            self._row_ring = [None] * self.RING

    # ------------------------------------------------------------------ setup
    def set_projector(self, group: int, weight: torch.Tensor, bias: torch.Tensor | None = None):
        """Projector of encoder group g: weight [d_llm, d_enc] bf16 (nn.Linear layout)."""
        assert self.projector
        assert weight.shape == (self.d_llm, self.d_enc[group]) and weight.dtype == torch.bfloat16
        self.weight[group] = weight.contiguous()
        self.bias[group] = None if bias is None else bias.contiguous()

    def cfg_for(self, table: StepTable):
        return make_cfg(table, self.capacity, self.gbs, self.dp, self.sp, self.world, 1,
                        self.method, self.pooled, self.rank,
                        row_bytes_in=tuple(2 * d for d in self.d_in),
                        row_bytes_ret=tuple(2 * d for d in self.d_ret), ret_mode=self.ret_mode,
                        row_bytes_grad=(2 * self.d_llm,) * N_GROUPS,
                        lssp_sp=self.lssp_sp if self.lssp_eta is not None else 0,
                        lssp_eta=self.lssp_eta or 0, reshard=self.reshard,
                        cp_threshold=self.cp_threshold, text_embed=self.text_embed,
                        chunk_bytes=self.chunk_bytes, reorder_group=self.reorder_group,
                        cost=self.cost)

    @property
    def llm(self) -> _Window:
        return self.llm_bufs[self.last_llm]

    def llm_view(self, rows: int | None = None) -> torch.Tensor:
        """Packed LLM input of this rank (with alternating buffers: the latest step's)."""
        n = self.max_llm_rows if rows is None else rows
        return self.llm.tensor[: n * self.d_llm * 2].view(torch.bfloat16).view(n, self.d_llm)

    def zero_llm(self):
        for b in self.llm_bufs:
            b.tensor.zero_()

    def recv_view(self, group: int, rows: int) -> torch.Tensor:
        d = self.d_in[group]
        return self.recv[group].tensor[: rows * d * 2].view(torch.bfloat16).view(rows, d)

    def enc_view(self, group: int, rows: int) -> torch.Tensor:
        d = self.d_ret[group]
        return self.enc_out[group][: rows * d].view(rows, d)

    # ------------------------------------------------------------------ stages
    def plan(self, dtab: DeviceTable, stream=None) -> Plan:
        """In-line plan into the single plan buffer (see plan_ahead for the ring)."""
        self.finish(stream)  # an overlapped projector may still read the buffer
        cfg = self.cfg_for(dtab.table)
        self._plan = plan_step(dtab, cfg, self._plan, stream)
        return self._plan

    # The plan of step k+1 needs only metadata, so it runs on a high-priority
    # side stream while step k's rows move.  RING plan buffers rotate: a plan
    # is read until its step's (possibly overlapped) projector finishes, so
    # with an overlapped projector two buffers would stall the planner.
    RING = 4

    def _ensure_ring(self):
        if self._ring is None:
            self._side = torch.cuda.Stream(self.device, priority=-1)
            self._ring = [None] * self.RING
            self._ready = [_event() for _ in range(self.RING)]
            self._freed = [None] * self.RING

    def plan_ahead(self, dtab: DeviceTable, slot: int, after=None) -> Plan:
        """Plan `dtab` into ring slot `slot` (0..RING-1) on the side stream.  `after`: an
        event the plan must follow (e.g. the step-table upload)."""
        self._ensure_ring()
        self.gemm_ctas = self._pipelined_gemm_ctas()
        side = self._side
        if self._freed[slot] is not None:
            side.wait_event(self._freed[slot])
        if after is not None:
            side.wait_event(after)
        cfg = self.cfg_for(dtab.table)
        p = self._ring[slot] = plan_step(dtab, cfg, self._ring[slot], side)
        if self.projector and not self.staged:
            # the GEMM's row map depends only on the plan: build it here, off the
            # step's critical path
            if self._row_ring[slot] is None:
                self._row_ring[slot] = torch.empty_like(self.row_dst)
            self._row_map(p, self._row_ring[slot], side)
        self._ready[slot].record(side)
        return p

    def _pipelined_gemm_ctas(self) -> int:
        """GEMM CTAs while the next step's plan runs beside it: all SMs when the
        planner's CTA fits next to a GEMM CTA (small step tables: its shared
        memory is a few KB), else one SM left free for it (MUX_GEMM_ALL_SMS)."""
        return self.num_sms if os.environ.get("MUX_GEMM_ALL_SMS", "0") == "1" \
            else self.num_sms - 1

    def run_pipeline(self, steps=None, *, n=None, prepare=None, encoder=None, after_step=None,
                     kernel_events=None, start_event=None, stream=None):
        """Run consecutive steps [(DeviceTable, arenas), ...] pipelined on `stream`.

        Streaming inputs: instead of `steps`, pass `n` and `prepare(k)` returning
        (DeviceTable, arenas, event or None); it is called once per step, one step
        ahead (before step k-1's work is issued), e.g. to upload step k from pinned
        host memory on a copy stream; the event orders the plan after that upload.

        The plan of step k+1 runs on the planner's side stream during step k;
        with overlap_dispatch, step k+1's dispatch also runs (copy stream) under
        step k's return, as soon as every rank signalled that step k's receive
        windows were consumed.  encoder(k, plan, stream) runs between a step's
        dispatch and its return (the encoder forward); after_step(k, plan,
        stream) after the return; `self.step_done` is then the event after which
        step k's plan and inputs are no longer read (with the staged projector
        it is on the projector stream: wait for it before reusing step k's input
        buffers).  kernel_events[k]: (start, end) events around step k's return
        kernel.  Without start_event the call is ordered after everything
        already enqueued on `stream`.  Raises RuntimeError when an earlier call
        left the path poisoned (a timed-out flag wait; see check_wait)."""
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.poll_status()
        if start_event is None:
            # order this call after everything already on `main` (inputs written
            # there, and an earlier call's encoder still reading the windows)
            start_event = _event()
            start_event.record(main)
        if steps is not None:
            n = len(steps)
            fixed = {k: (steps[k][0], steps[k][1], None) for k in range(n)}
            get = fixed.__getitem__
        else:
            cache: dict = {}

            def get(k):
                if k not in cache:
                    cache[k] = prepare(k)
                return cache[k]
        R = self.RING
        if not n:
            return
        self._ensure_ring()
        base = getattr(self, "_kstep", 0)
        slot = [(base + k) % R for k in range(n)]
        ov = self.overlap_dispatch
        d0, a0, e0 = get(0)
        if e0 is not None and start_event is not None:
            self._side.wait_event(start_event)
        self.plan_ahead(d0, slot[0], after=e0 if e0 is not None else start_event)
        if ov:
            if getattr(self, "_copy", None) is None:
                self._copy = torch.cuda.Stream(self.device)
                self._dispatched = [_event() for _ in range(R)]
            cs = self._copy
            cs.wait_event(self._ready[slot[0]])
            # waits for every peer's last "consumed" signal of an earlier call too
            self.dispatch_overlapped(self._ring[slot[0]], a0, cs)
            self._dispatched[slot[0]].record(cs)
        for k in range(n):
            s = slot[k]
            if k + 1 < n:
                dn, _, en = get(k + 1)
                self.plan_ahead(dn, slot[k + 1], after=en)
            p = self._ring[s]
            if ov:
                main.wait_event(self._dispatched[s])
            else:
                main.wait_event(self._ready[s])
                self.dispatch(p, get(k)[1], main)
            if encoder is not None:
                encoder(k, p, main)
            if ov:
                self.signal_consumed(main, fuse=True)
                ev = _event()
                ev.record(main)
            self.kernel_events = kernel_events[k] if kernel_events else None
            self._freed[s] = self.return_scatter(p, main)
            self.kernel_events = None
            if ov and k + 1 < n:
                # issued after the return kernel: the copy stream's spin-wait for
                # every rank's "consumed" signal (carried by that kernel) must never
                # sit in front of it in a shared hardware queue
                cs.wait_event(self._ready[slot[k + 1]])
                self.dispatch_overlapped(self._ring[slot[k + 1]], get(k + 1)[1], cs, after=ev)
                self._dispatched[slot[k + 1]].record(cs)
            self.step_done = self._freed[s]
            if after_step is not None:
                after_step(k, p, main)
            if steps is None:  # streaming: step k's inputs are issued; drop them
                cache.pop(k, None)
        self._kstep = base + n
        if self._status_host is not None:  # async status mirror, raised at the next call
            self._status_host.copy_(self.wait_err, non_blocking=True)
            self._status_ev = _event()
            self._status_ev.record(main)

    def _arena_table(self, arenas) -> torch.Tensor:
        """Device table of loader-arena pointers, cached per arena set (no sync
        once warm)."""
        key = tuple(int(a.data_ptr()) if a is not None else 0 for a in arenas)
        t = self._arena_tables.get(key)
        if t is None:
            t = _ptr_table(key, self.device)
            self._arena_tables[key] = t
        return t

    def _exchange(self, plan: Plan, which: int, src, dst, stream):
        """One segment-copy exchange; across GPUs the last CTA signals every
        peer and a flag wait orders the stream after every peer's copy."""
        L = _lib.lib()
        s = _stream_ptr(stream)
        ke = self.kernel_events if which == 1 else None
        if ke is not None:
            ke[0].record(stream if stream is not None else torch.cuda.current_stream(self.device))
        if self.world == 1:
            _lib.check(L.mux_segcopy(C.byref(plan.cfg), plan.ptr, which, src.data_ptr(),
                                     dst.data_ptr(),
                                     self.dispatch_grid if which == 0 else self.copy_grid,
                                     self.sync[2 * which:].data_ptr(), s), "mux_segcopy")
            if ke is not None:
                ke[1].record(stream if stream is not None else
                             torch.cuda.current_stream(self.device))
            return
        # beside an overlapped projector (which holds shared memory) copy CTAs stay lean
        grid = -2 * self.num_sms if self.staged else \
            (self.dispatch_grid if which == 0 else self.copy_grid)
        fptrs, flags, epoch = (self.flag_ptrs_d, self.flags_d, self.epoch_d) if which == 0 else \
            (self.flag_ptrs, self.flags, self.epoch_ctr)
        _lib.check(L.mux_segcopy_ex(C.byref(plan.cfg), plan.ptr, which, src.data_ptr(),
                                    dst.data_ptr(), grid, -1, fptrs.data_ptr(),
                                    self.sync[2 * which:].data_ptr(), epoch.data_ptr(),
                                    self.wait_err.data_ptr(), s), "mux_segcopy_ex")
        if ke is not None:
            ke[1].record(stream if stream is not None else torch.cuda.current_stream(self.device))
        _lib.check(L.mux_wait(self.world, flags.tensor.data_ptr(), epoch.data_ptr(),
                              self.timeout_ms, self.wait_err.data_ptr(), s), "mux_wait")

    def dispatch(self, plan: Plan, arenas, stream=None):
        """Pack + dispatch: loader rows of every group to their encoder rank."""
        self._exchange(plan, 0, self._arena_table(arenas), self.recv_dst, stream)

    def signal_consumed(self, stream=None, fuse: bool = False):
        """This rank's encoder has read its receive windows (E channel): peers may
        push the next step's rows (dispatch_overlapped).  fuse=True: the next
        return_scatter's projector GEMM carries the signal at its start instead
        of a separate launch."""
        if self.world == 1:
            return
        self._e_sent += 1
        if fuse and self.projector and not self.staged and \
                os.environ.get("MUX_FUSE_E", "1") != "0":
            self._fuse_e = True
            return
        # a permission, not data: no system fence (mux_signal_ex)
        _lib.check(_lib.lib().mux_signal_ex(self.rank, self.world, self.flag_ptrs_e.data_ptr(),
                                            self.epoch_e.data_ptr(), 0, _stream_ptr(stream)),
                   "mux_signal_ex")

    def dispatch_overlapped(self, plan: Plan, arenas, stream, after=None):
        """The next step's dispatch on its own `stream`, under the current step's
        return: waits (on `stream`) for `after` (this rank's signal_consumed) and
        for every peer's signal_consumed, then pushes.  Needs overlap_dispatch=True
        (alternating LLM buffers keep the returns of consecutive steps apart)."""
        if not self.overlap_dispatch:
            raise ValueError("MuxPath(overlap_dispatch=True) is needed")
        if after is not None:
            stream.wait_event(after)
        if self.world > 1:  # every peer's E count reaches mine (host-known target)
            _lib.check(_lib.lib().mux_wait_value(self.world, self.flags_e.tensor.data_ptr(),
                                                 self._e_sent, self.timeout_ms,
                                                 self.wait_err.data_ptr(), _stream_ptr(stream)),
                       "mux_wait_value")
        self.dispatch(plan, arenas, stream)

    def encode_standin(self, plan: Plan, dtab: DeviceTable, stream=None):
        """Deterministic encoder stand-in E(id, t, c) into the encoder output."""
        L = _lib.lib()
        for g in range(N_GROUPS):
            _lib.check(L.mux_encoder_standin(C.byref(plan.cfg), plan.ptr, dtab.ids, dtab.lens, g,
                                             self.d_ret[g], self.enc_out[g].data_ptr(),
                                             _stream_ptr(stream)), "mux_encoder_standin")

    def return_scatter(self, plan: Plan, stream=None) -> torch.cuda.Event:
        """Return + scatter (projector off) or projector + scatter (on).

        Returns the event after which `plan` is no longer read and this step's
        LLM rows are final.  No host synchronisation: row counts come from the
        plan header on the device."""
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        if not self.staged:  # alternate LLM buffers when there are two
            self.last_llm = self._nret % len(self.llm_bufs)
            self._nret += 1
        if not self.projector:
            self._exchange(plan, 1, self.enc_src, self.llm_dst[self.last_llm], main)
        elif self.staged:
            return self._return_staged(plan, main)
        else:
            self._project(plan, main)
        ev = _event()
        ev.record(main)
        return ev

    def _row_map(self, plan: Plan, row_dst: torch.Tensor, stream):
        """row_dst[g * max_rows + m] = (rank << 40) | row of encoder row m of group g."""
        _lib.check(_lib.lib().mux_return_rows(C.byref(plan.cfg), plan.ptr, -1,
                                              row_dst.data_ptr(), self.max_rows,
                                              _stream_ptr(stream)), "mux_return_rows")
        plan.row_map = row_dst

    def _project(self, plan: Plan, main):
        """GEMM on this (encoder) rank, every group in one launch; the epilogue
        stores every row at its (rank, row), on this GPU or an NVLink peer."""
        L = _lib.lib()
        s = _stream_ptr(main)
        hdr = plan.ptr + plan.layout.header
        rmap = getattr(plan, "row_map", None)
        if rmap is None:
            self._row_map(plan, self.row_dst, main)
            rmap = self.row_dst
        groups = (_lib.ProjGroup * N_GROUPS)()
        n = 0
        for g in range(N_GROUPS):
            if self.weight[g] is None:
                continue
            b = self.bias[g]
            groups[n] = _lib.ProjGroup(
                self.enc_out[g].data_ptr(), self.weight[g].data_ptr(),
                0 if b is None else b.data_ptr(), self.max_rows,
                hdr + 8 * (_lib.H_RECV_ROWS0 + g), self.d_enc[g], 0,
                rmap.data_ptr() + 8 * g * self.max_rows)
            n += 1
        plan.row_map = None  # consumed; the next plan in this slot rebuilds it
        ke = self.kernel_events
        if ke is not None:
            ke[0].record(main)
        if self.world == 1:
            _lib.check(L.mux_proj_scatter_grouped(groups, n, self.d_llm,
                                                  self.llm_dst[self.last_llm].data_ptr(),
                                                  self.gemm_ctas, s),
                       "mux_proj_scatter_grouped")
        else:  # the GEMM's last CTA signals every peer (+ a pending E signal at its start)
            fe = self._fuse_e
            self._fuse_e = False
            _lib.check(L.mux_proj_scatter_grouped_signal(
                groups, n, self.d_llm, self.llm_dst[self.last_llm].data_ptr(), self.gemm_ctas,
                self.rank,
                self.world, self.flag_ptrs.data_ptr(), self.sync[6:].data_ptr(),
                self.epoch_ctr.data_ptr(), self.flag_ptrs_e.data_ptr() if fe else None,
                self.epoch_e.data_ptr() if fe else None, self.wait_err.data_ptr(), s),
                "mux_proj_scatter_grouped_signal")
        if ke is not None:
            ke[1].record(main)
        if self.world > 1:
            _lib.check(L.mux_wait(self.world, self.flags.tensor.data_ptr(),
                                  self.epoch_ctr.data_ptr(), self.timeout_ms,
                                  self.wait_err.data_ptr(), s), "mux_wait")

    def _return_staged(self, plan: Plan, main) -> torch.cuda.Event:
        """d_enc rows -> the owner's staging window (main-stream exchange), then
        the owner's GEMM on the projector stream, overlapped with what follows."""
        L = _lib.lib()
        b = self._kret % 2
        self._kret += 1
        if self._ev_p[b] is not None:  # the projector of step k-2 has read stage[b]
            main.wait_event(self._ev_p[b])
        self._exchange(plan, 1, self.enc_src, self.stage_dst[b], main)
        ev_r = _event()
        ev_r.record(main)
        proj = self._proj
        proj.wait_event(ev_r)
        s = _stream_ptr(proj)
        hdr = plan.ptr + plan.layout.header
        rd = self.row_dst_b[b]
        for g in range(N_GROUPS):
            if self.weight[g] is None:
                continue
            _lib.check(L.mux_stage_rows(C.byref(plan.cfg), plan.ptr, plan.lens_ptr, g,
                                        rd.data_ptr(), self.max_llm_rows, s), "mux_stage_rows")
            bias = self.bias[g]
            _lib.check(L.mux_proj_scatter_dev(
                self.stage[b][g].tensor.data_ptr(), self.weight[g].data_ptr(),
                0 if bias is None else bias.data_ptr(), self.max_llm_rows,
                hdr + 8 * (_lib.H_STAGE_ROWS0 + g), self.d_enc[g], self.d_llm,
                rd.data_ptr(), self.llm_dst[b].data_ptr(), self.gemm_ctas, s),
                "mux_proj_scatter_dev")
        ev_p = _event(timing=True)
        ev_p.record(proj)
        self._ev_p[b] = ev_p
        self.last_llm = b
        return ev_p

    # ------------------------------------------------------------- text rows
    def embed_text(self, plan: Plan, tokens: torch.Tensor, table: torch.Tensor, stream=None):
        """Text rows of this rank's packed LLM input: row <- table[token id] for
        every text token this rank owns (needs text_embed=True).
        tokens: int32 ids of the step's text samples in table order (device);
        table: bf16 [vocab, d_llm] embedding rows (device, replicated)."""
        if not self.text_embed:
            raise ValueError("MuxPath(text_embed=True) is needed for embed_text")
        assert tokens.dtype == torch.int32 and table.dtype == torch.bfloat16
        assert table.shape[1] == self.d_llm and table.is_contiguous()
        if getattr(self, "text_err", None) is None:
            self.text_err = torch.zeros(1, dtype=torch.int32, device=self.device)
        _lib.check(_lib.lib().mux_text_embed(
            C.byref(plan.cfg), plan.ptr, tokens.data_ptr(), table.data_ptr(), table.shape[0],
            self.d_llm, self.llm.tensor.data_ptr(), self.text_err.data_ptr(),
            _stream_ptr(stream)), "mux_text_embed")

    def check_text(self):
        """Raise if any token id was outside the embedding table (synchronises)."""
        if getattr(self, "text_err", None) is not None and int(self.text_err.item()):
            raise ValueError(f"{int(self.text_err.item())} text rows had token ids outside "
                             "the embedding table")

    # --------------------------------------------------------- gradient return
    def _ensure_grad(self):
        if getattr(self, "grad", None) is None:
            dev, w = self.device, self.world
            width = self.d_llm  # dL/d(projector output or returned rows): d_llm wide
            self.grad = [_Window(self.max_rows * width * 2, dev, self.group, w)
                         for _ in range(N_GROUPS)]
            self.grad_dst = _ptr_table([self.grad[g].ptrs[r] for r in range(w)
                                        for g in range(N_GROUPS)], dev)
            self._dy_tables: dict = {}
            if w > 1:
                torch.cuda.synchronize()
                self.flags.handle.barrier()

    def grad_return(self, plan: Plan, dy: torch.Tensor, stream=None):
        """Backward of return + scatter (restore_order on the
        gradient path): this rank's dY rows at the placeholder positions of its
        packed LLM input go back to the encoder ranks, in encoder order, into
        `grad_view(g, rows)`.  dy: [>= llm rows, d_llm] bf16 on this GPU.
        With the projector, dX = dY W and dW = dY^T X then run on the encoder
        rank (`projector_backward`)."""
        if self.ret_mode != _lib.RET_FINAL:
            raise ValueError("gradient return is defined for the final-row layouts")
        assert dy.dtype == torch.bfloat16 and dy.shape[-1] == self.d_llm and dy.is_contiguous()
        self._ensure_grad()
        key = dy.data_ptr()
        t = self._dy_tables.get(key)
        if t is None:
            t = _ptr_table([key] * N_GROUPS, self.device)
            self._dy_tables[key] = t
        self._exchange(plan, 2, t, self.grad_dst, stream)

    def projector_backward(self, group: int, rows: int | None = None,
                           x: torch.Tensor | None = None, plan: Plan | None = None,
                           stream=None, want=("dx", "dw", "db")):
        """dX = G W, dW = G^T X and db = sum_m G[m, :] for encoder group `group`
        on this encoder rank (SPEC.md:411 gradient path; tcgen05 CTA-pair GEMMs
        of csrc/proj_bwd.cu: dX on the forward kernel with W^T, dW with MN-major
        operands and db fused into it).  G = the returned gradient rows in
        encoder order (`grad_return`, `grad_view`); x = the projector input
        [>= rows, d_enc] (default: this rank's encoder output).  The row count
        is `rows` (host) or, with `plan`, read on the device (no sync).  Rows
        [M, round_up(M, 64)) of G and x are zeroed.  Returns (dx [M or max rows,
        d_enc], dw [d_llm, d_enc], db [d_llm]) bf16, None for products not in
        `want`."""
        assert self.projector and self.weight[group] is not None
        self._ensure_grad()
        dev, L = self.device, _lib.lib()
        K, N = self.d_enc[group], self.d_llm
        X = self.enc_out[group].view(-1, K) if x is None else x
        assert X.dtype == torch.bfloat16 and X.is_contiguous() and X.shape[1] == K
        m_max = min(self.max_rows, X.shape[0])
        if plan is not None:
            m_dev = plan.ptr + plan.layout.header + 8 * (_lib.H_RECV_ROWS0 + group)
        else:
            if rows is None or rows > m_max:
                raise ValueError(f"rows {rows} must be given and <= {m_max}")
            m_dev = 0
            m_max = rows
        G = self.grad[group].tensor[: self.max_rows * N * 2].view(torch.bfloat16).view(-1, N)
        ws_need = L.mux_proj_backward_workspace(K, N, self.num_sms)
        ws = getattr(self, "_bwd_ws", None)
        if ws is None or ws.numel() < ws_need:
            ws = self._bwd_ws = torch.empty(ws_need, dtype=torch.uint8, device=dev)
        dx = torch.empty(max(m_max, 1), K, dtype=torch.bfloat16, device=dev) \
            if "dx" in want else None
        dw = torch.empty(N, K, dtype=torch.bfloat16, device=dev) if "dw" in want else None
        db = torch.empty(N, dtype=torch.bfloat16, device=dev) if "db" in want else None
        _lib.check(L.mux_proj_backward(
            G.data_ptr(), X.data_ptr(), self.weight[group].data_ptr(), m_max, m_dev or None, K,
            N, dx.data_ptr() if dx is not None else None,
            dw.data_ptr() if dw is not None else None, db.data_ptr() if db is not None else None,
            ws.data_ptr(), ws.numel(), self.num_sms, _stream_ptr(stream)), "mux_proj_backward")
        if dx is not None and plan is None:
            dx = dx[:rows]
        return dx, dw, db

    def grad_view(self, group: int, rows: int) -> torch.Tensor:
        self._ensure_grad()
        return self.grad[group].tensor[: rows * self.d_llm * 2].view(torch.bfloat16).view(
            rows, self.d_llm)

    def finish(self, stream=None):
        """Make `stream` wait for every outstanding overlapped projector."""
        if self.staged:
            main = stream if stream is not None else torch.cuda.current_stream(self.device)
            for ev in self._ev_p:
                if ev is not None:
                    main.wait_event(ev)

    # ------------------------------------------------------------ CUDA graphs
    def capture_steps(self, dtabs, arenas_list):
        """One CUDA graph per distinct step i: (plan of step i+1 on the side
        stream) overlapped with (dispatch + return/scatter of step i).  Replay
        with `StepGraphs.replay(k)`; every kernel of the pipelined step is a
        graph node, so the host issues one launch per step."""
        return StepGraphs(self, dtabs, arenas_list)

    _POISON_WHY = {1: "a cross-GPU completion flag wait timed out",
                   2: "a peer rank's step was poisoned (its flag wait timed out)"}

    def _raise_status(self, code: int):
        raise RuntimeError(f"data path poisoned: {self._POISON_WHY.get(code, code)}; the "
                           "exchange buffers of this and later steps are not valid (every "
                           "rank calls reset_status() to recover)")

    def check_wait(self):
        """Synchronise and raise if the path is poisoned."""
        code = int(self.wait_err.item())
        if code:
            self._raise_status(code)

    def reset_status(self):
        """Collective recovery from a poisoned path (every rank calls it): drain
        this GPU, clear the status word, every flag channel and epoch counter and
        the copy counters, then barrier.  Buffers keep their (partial) contents;
        the next step rewrites them."""
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)
        self.wait_err.zero_()
        for f in (self.flags, self.flags_d, self.flags_e):
            f.tensor.zero_()
        for e in (self.epoch_ctr, self.epoch_d, self.epoch_e):
            e.zero_()
        self.sync.zero_()
        self._e_sent = 0
        self._fuse_e = False
        self._status_ev = None
        if self._status_host is not None:
            self._status_host.zero_()
        torch.cuda.synchronize(self.device)
        if self.world > 1:  # every rank's flags are clear before anyone signals again
            self.flags.handle.barrier()

    def poll_status(self):
        """Raise if an earlier run_pipeline's status copy has landed and shows a
        poisoned path (no synchronisation)."""
        ev = self._status_ev
        if ev is not None and ev.query():
            self._status_ev = None
            code = int(self._status_host[0])
            if code:
                self._raise_status(code)


class StepGraphs:
    """Captured pipelined steps (see MuxPath.capture_steps)."""

    def __init__(self, path: MuxPath, dtabs, arenas_list):
        n = len(dtabs)
        if n % 2:
            raise ValueError("capture an even number of distinct steps (two plan buffers)")
        path._ensure_ring()
        path.gemm_ctas = path._pipelined_gemm_ctas()
        dev = path.device
        self.path, self.n = path, n
        cfgs = [path.cfg_for(d.table) for d in dtabs]
        biggest = max(layout_of(c).total for c in cfgs)
        self.blobs = [torch.zeros(biggest, dtype=torch.uint8, device=dev) for _ in range(2)]
        plans = [Plan(cfgs[i], dev, self.blobs[i % 2]) for i in range(n)]
        self.plans = plans
        side = path._side
        # eager pass: caches pointer tables / kernel attributes, checks every plan
        for i in range(n):
            plan_step(dtabs[i], cfgs[i], plans[i])
            plans[i].check(dtabs[i].table)
            path.dispatch(plans[i], arenas_list[i])
            path.return_scatter(plans[i])
        torch.cuda.synchronize(dev)
        self.graphs = []
        cap = torch.cuda.Stream(dev)
        for i in range(n):
            j = (i + 1) % n
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                main = torch.cuda.current_stream(dev)
                side.wait_stream(main)
                plan_step(dtabs[j], cfgs[j], plans[j], side)
                path.dispatch(plans[i], arenas_list[i], main)
                path.return_scatter(plans[i], main)
                path.finish(main)
                main.wait_stream(side)
            self.graphs.append(g)
        self.dtabs, self.cfgs = dtabs, cfgs

    def prime(self, k: int, stream=None):
        """Plan step k (each graph plans step i+1 while running step i), so a
        replay sequence starting at k must be primed with step k's plan."""
        i = k % self.n
        plan_step(self.dtabs[i], self.cfgs[i], self.plans[i], stream)

    def replay(self, k: int):
        self.graphs[k % self.n].replay()
