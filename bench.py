"""Benchmark of the per-step encoder<->LLM data path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2|target1|cfg5|...]
                    [--impl ours|reference]

One step = plan (FFD + batch + LPT rebalance + reshard geometry, on device)
-> pack + dispatch (push over NVLink at N > 1) -> return + scatter into the
packed LLM input (projector GEMM fused with the scatter for cfg2).  The
encoder itself is out of scope: its output buffer is filled once by the
deterministic stand-in before timing.  Inputs are synthetic (the reference's
own generator, restated in workload.py) and resident in HBM for `value`; `e2e`
runs the same step through the public API from pinned host buffers.

Steps are pipelined (MuxPath.run_pipeline): the plan of step k+1 runs on a
side stream and, with the default --pipeline 2, its dispatch on a copy stream
under step k's projector/return; the timed region covers K whole steps.

Weak scaling: every GPU owns `gbs_per_replica` sequences (dp = N).
Rank 0 prints one JSON line.  Tuning switches (env and build macros, with their
defaults and measurements): DESIGN.md §11.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=os.environ.get("MUX_BENCH_CONFIG", "cfg2"))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--distinct", type=int, default=8, help="distinct step inputs cycled")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-nested", action="store_true",
                    help="skip the nested north-star record (target1 at 1 GPU, cfg5 at N>1)")
    ap.add_argument("--no-comparator", action="store_true",
                    help="skip the cuBLAS + index_copy_ comparator of the projector")
    ap.add_argument("--stages", action="store_true", help="per-stage timing breakdown")
    ap.add_argument("--pipeline", type=int, default=2,
                    help="1: plan step k+1 on a side stream during step k; 2 (default): also "
                         "dispatch step k+1 under step k's return")
    ap.add_argument("--method", default="lpt_local",
                    choices=["lpt", "kk", "lpt_local", "lpt_local_rw"],
                    help="encoder balancing: locality-first LPT (default), LPT or KK")
    ap.add_argument("--hang-dump", type=float, default=0.0,
                    help="dump Python stacks after this many seconds (debug)")
    ap.add_argument("--lssp-eta", type=int, default=-1,
                    help="LSSP eta split: samples longer than this are encoded as token "
                         "shards over encoder groups (-1: off)")
    ap.add_argument("--lssp-sp", type=int, default=0, help="LSSP group size (0: all ranks)")
    ap.add_argument("--reshard", default="ulysses", choices=["ulysses", "cp_hybrid"],
                    help="LLM placement over each replica's sp ranks")
    ap.add_argument("--cp-threshold", type=int, default=0, help="CpHybrid threshold (0: C/sp)")
    ap.add_argument("--text-embed", action="store_true",
                    help="also gather the text tokens' embedding rows into the packed LLM "
                         "input every step (SURVEY §8f-4)")
    ap.add_argument("--graphs", type=int, default=0,
                    help="1: replay one captured CUDA graph per pipelined step")
    return ap.parse_args()


# ----------------------------------------------------------------------------
# workload
# ----------------------------------------------------------------------------

def balance_summary(plans_info, steps_idx):
    """Balance diagnostics per step: encoder rows per rank before
    the reorder (by origin rank) and after it (by encoder rank), and max/mean
    imbalance ratios, averaged over the timed steps (first step's vectors kept)."""
    def imb(v):
        v = np.asarray(v, np.float64)
        return float(v.max() / v.mean()) if v.size and v.mean() > 0 else 1.0
    first = plans_info[steps_idx[0]]
    return {"pre_loads_first_step": first["pre"].tolist(),
            "post_loads_first_step": first["post"].tolist(),
            "pre_imbalance": float(np.mean([imb(plans_info[i]["pre"]) for i in steps_idx])),
            "post_imbalance": float(np.mean([imb(plans_info[i]["post"]) for i in steps_idx])),
            "unit": "encoder rows (modality tokens) per rank; imbalance = max / mean"}


def exchange_summary(plans_info, steps_idx, rank):
    """Rank-local bytes per step of the two exchanges and the share leaving the
    GPU over NVLink (the rest is a local HBM copy)."""
    n = len(steps_idx)
    avg = {k: sum(plans_info[i][k] for i in steps_idx) / n
           for k in ("disp_bytes", "disp_remote", "ret_bytes", "ret_remote")}
    return {"rank": rank, "dispatch_bytes": avg["disp_bytes"],
            "dispatch_remote_frac": avg["disp_remote"] / max(avg["disp_bytes"], 1),
            "return_bytes": avg["ret_bytes"],
            "return_remote_frac": avg["ret_remote"] / max(avg["ret_bytes"], 1)}


def workload(name, world):
    from paper_2605_08962_b200 import configs
    cfg = dict(configs.CONFIGS[name])
    sp = cfg["sp"] if world % cfg["sp"] == 0 and world >= cfg["sp"] else 1
    dp = world // sp
    gbs = cfg["gbs_per_replica"] * dp
    return cfg, dp, sp, gbs


def generate_steps(name, world, n_steps):
    """Host generation of n chained steps with the reference's generator
    (workload.generate_batch's draw loop; hybrid_pack on the GPU)."""
    from paper_2605_08962_b200 import configs, workload as W
    from paper_2605_08962_b200.planner import StepTable
    cfg, dp, sp, gbs = workload(name, world)
    reg, sched = configs.build(W, name)
    carry, modality_of, out = None, {}, []
    for step in range(n_steps):
        seqs, chunks = W.draw_step_chunks(reg, sched, step, cfg["seed"], gbs, configs.CAPACITY,
                                          carry if cfg["carry"] else None)
        for ch in chunks:
            for s in ch:
                modality_of[s.id] = s.modality
        table = StepTable.from_chunks(list(carry or []) if cfg["carry"] else [], chunks,
                                      modality_of)
        out.append(table)
        carry = seqs[gbs:]
    return out


# ----------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------

def _clock_proc(index, q, stop, period):
    """Child process: sample SM clock / throttle reasons until `stop` is set."""
    reasons = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
    sm, seen, mx, src = [], set(), None, "nvml"
    try:
        import pynvml as n
        n.nvmlInit()
        h = n.nvmlDeviceGetHandleByIndex(index)
        mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
        q.put("ready")
        while not stop.is_set():
            sm.append(n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM))
            r = n.nvmlDeviceGetCurrentClocksEventReasons(h)
            seen.update(k for k, b in reasons.items() if r & b)
            time.sleep(period)
    except Exception as e:  # no NVML: nvidia-smi polling
        src = f"nvidia-smi ({type(e).__name__})"
        try:
            q.put("ready")
        except Exception:
            pass
        qq = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not stop.is_set():
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(index), f"--query-gpu={qq}",
                                    "--format=csv,noheader,nounits"], capture_output=True,
                                   text=True, timeout=5)
                f = [x.strip() for x in r.stdout.strip().split(",")]
                sm.append(float(f[0]))
                mx = float(f[1])
                seen.update(nm for k, nm in enumerate(names)
                            if f[2 + k].lower().startswith("active"))
            except Exception:
                pass
            time.sleep(0.05)
    q.put({"sm": sm, "mx": mx, "reasons": sorted(seen), "source": src})


class Clocks:
    """SM clocks and throttle reasons sampled by a child process (no GIL
    contention with the launch loop) from before warm-up to the end of the
    timed region."""

    def __init__(self, index, period=0.001):
        import multiprocessing as mp
        ctx = mp.get_context("spawn")
        self.q, self.stop = ctx.Queue(), ctx.Event()
        self.p = ctx.Process(target=_clock_proc, args=(index, self.q, self.stop, period),
                             daemon=True)
        self.res = None

    def __enter__(self):
        self.p.start()
        try:
            self.q.get(timeout=60)
        except Exception:
            pass
        return self

    def __exit__(self, *a):
        self.stop.set()
        try:
            self.res = self.q.get(timeout=30)
        except Exception:
            self.res = None
        self.p.join(timeout=10)

    def summary(self):
        r = self.res
        if not r or not r["sm"]:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"],
                    "samples": 0}
        return {"sm_mhz": float(np.median(r["sm"])), "sm_min_mhz": float(min(r["sm"])),
                "sm_max_mhz": float(r["mx"]) if r["mx"] else None, "reasons": r["reasons"],
                "samples": len(r["sm"]), "source": r["source"],
                "window": "warm-up + 100 ms soak + timed region"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p["bf16_tflops_sustained"]), \
            "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------

def choose_tensor_peak(clocks):
    """Burst or sustained bf16 denominator from the run's own clock record:
    sustained only when the GPU was power-capped (sw_power_cap seen) or its
    median SM clock sat below 0.9x max; otherwise the burst figure."""
    hbm, burst, sus, src = peaks()
    reasons = (clocks or {}).get("reasons") or []
    med, mx = (clocks or {}).get("sm_mhz"), (clocks or {}).get("sm_max_mhz")
    capped = "sw_power_cap" in reasons or (med is not None and mx and med < 0.9 * mx)
    if capped:
        return sus, (f"bf16_tflops_sustained ({src}): sw_power_cap or median clock < 0.9x max "
                     f"in this run's record; burst {burst}")
    return burst, (f"bf16_tflops burst ({src}): median clock {med} of max {mx} MHz, no power "
                   f"cap in this run's record; sustained {sus}")


def config_dict(name, world, n_distinct, M_per_step, T_per_step):
    """The `config` both arms print (identical for the same flags)."""
    from paper_2605_08962_b200 import configs
    cfg, dp, sp, gbs = workload(name, world)
    return {"workload": name, "global_batch": gbs, "seq_len": configs.CAPACITY,
            "parallelism": f"enc dp{world} / llm dp{dp} sp{sp}",
            "projector": bool(cfg["projector"]), "d_in": list(configs.D_IN),
            "d_enc": list(configs.D_ENC), "d_llm": configs.D_LLM,
            "distinct_steps": n_distinct, "modality_tokens_per_step": M_per_step,
            "llm_tokens_per_step": T_per_step,
            "l2": "per-step working set > 126 MB L2 (inputs larger than L2)"}


def n_distinct_of(args):
    return max(1, min(args.distinct, args.steps + args.warmup))


def timed_indices(args, n_distinct):
    return [(args.warmup + k) % n_distinct for k in range(args.steps)]


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_08962_b200 import _lib, build as B

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N>1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    if not os.path.exists(B.LIB):
        if rank == 0:
            B.build()
        if world > 1:
            dist.barrier()
    _lib.lib()
    ctx = dict(world=world, rank=rank, local=local, dev=dev, group=group)

    line = measure(args.config, args, ctx, primary=True)
    # the north-star records beside the headline, in the same process: target-1
    # (projector off, bit-exact, HBM roofline) at one GPU; the phase-cycling
    # mixed batch (projector off, NVLink roofline) across GPUs
    if not args.no_nested:
        nested = "target1" if world == 1 else "cfg5"
        if nested != args.config:
            sub = measure(nested, args, ctx, primary=False)
            for k in ("metric", "unit", "higher_is_better", "dtype", "data", "vs_baseline",
                      "n_gpus", "steps", "warmup", "scaling"):
                sub.pop(k, None)
            line[nested] = sub
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def measure(name, args, ctx, primary=True):
    """One workload through the pipelined step loop; returns its JSON record."""
    import torch
    import torch.distributed as dist

    from paper_2605_08962_b200 import _lib, configs
    from paper_2605_08962_b200.dataplane import MuxPath
    from paper_2605_08962_b200.planner import DeviceTable

    world, rank, local, dev, group = (ctx[k] for k in ("world", "rank", "local", "dev", "group"))
    cfg, dp, sp, gbs = workload(name, world)
    projector = bool(cfg["projector"])
    d_in, d_enc, d_llm = configs.D_IN, configs.D_ENC, configs.D_LLM
    n_distinct = n_distinct_of(args)
    tables = generate_steps(name, world, n_distinct)

    path = MuxPath(capacity=configs.CAPACITY, gbs=gbs, dp=dp, sp=sp, world=world, rank=rank,
                   d_in=d_in, d_enc=d_enc, d_llm=d_llm, projector=projector, device=dev,
                   group=group, method=args.method,
                   lssp_eta=args.lssp_eta if args.lssp_eta >= 0 else None,
                   lssp_sp=args.lssp_sp or world, reshard=args.reshard,
                   cp_threshold=args.cp_threshold, overlap_dispatch=args.pipeline >= 2,
                   text_embed=args.text_embed)
    if projector:
        gen = torch.Generator(device=dev).manual_seed(77)
        for g in range(2):
            w = (torch.randn(d_llm, d_enc[g], device=dev, generator=gen) / d_enc[g] ** 0.5)
            path.set_projector(g, w.to(torch.bfloat16),
                               torch.randn(d_llm, device=dev, generator=gen).to(torch.bfloat16))

    # device-resident inputs: one step table + loader arenas per distinct step
    dtabs, arenas, plans_info = [], [], []
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    for t in tables:
        dt = DeviceTable(t, dev)
        plan = path.plan(dt)
        h = plan.check(t)
        info = plan.host()
        ar = [torch.randn(max(int(info["arena_rows"][rank, g]), 1), d_in[g], device=dev,
                          generator=gen).to(torch.bfloat16) for g in range(2)]
        dtabs.append(dt)
        arenas.append(ar)
        # return bytes of this rank per destination rank (NVLink accounting)
        ret_to = np.zeros(world)  # bytes that cross to each rank: with the fused projector
        for (_s, _d, rows, g, r) in info["rseg"]:  # the GEMM stores d_llm-wide rows
            wide = d_llm if (projector and not path.staged) else path.d_ret[int(g)]
            ret_to[int(r)] += int(rows) * 2 * wide
        disp_to = np.zeros(world)
        for (_s, _d, rows, g, r) in info["dseg"]:
            disp_to[int(r)] += int(rows) * 2 * d_in[int(g)]
        m_tokens = int(info["recv_rows"].sum())  # modality tokens of the whole batch
        pre = info["arena_rows"].sum(1).astype(np.float64)   # rows per origin (loader) rank
        post = info["recv_rows"].sum(1).astype(np.float64)   # rows per encoder rank
        plans_info.append(dict(M=m_tokens, T=int(info["llm_rows"].sum()),
                               S=int(h[_lib.H_N_BATCH]),
                               recv=(int(h[_lib.H_RECV_ROWS0]), int(h[_lib.H_RECV_ROWS1])),
                               disp_bytes=int(h[_lib.H_DISPATCH_BYTES]),
                               ret_bytes=int(h[_lib.H_RETURN_BYTES]),
                               disp_remote=int(h[_lib.H_DISPATCH_REMOTE]),
                               ret_remote=int(h[_lib.H_RETURN_REMOTE]),
                               ret_to=ret_to, disp_to=disp_to, pre=pre, post=post))
    text_tokens, text_table = [], None
    if args.text_embed:  # synthetic token ids per distinct step, a 32K-row embedding table
        text_table = torch.randn(32000, d_llm, device=dev).to(torch.bfloat16)
        for t in tables:
            n_text = int(sum(int(L) for L, m in zip(t.lens, t.mods) if m == 0))
            text_tokens.append(torch.randint(0, 32000, (max(n_text, 1),), device=dev,
                                             dtype=torch.int32))
    # encoder output: the stand-in fills it once (encoder compute is out of scope)
    plan = path.plan(dtabs[0])
    path.encode_standin(plan, dtabs[0])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    stream = torch.cuda.current_stream()
    ev_dom = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]

    def one_step(k, timed_dom=None):
        i = k % n_distinct
        p = path.plan(dtabs[i], stream)
        path.dispatch(p, arenas[i], stream)
        path.kernel_events = timed_dom  # around the return kernel itself
        path.return_scatter(p, stream)
        path.kernel_events = None

    def run_steps(k0, n, timed_dom=None, start_ev=None):
        """n steps from k0; with --pipeline the plan of step k+1 runs on the side
        stream during step k (every plan stays inside the window)."""
        if graphs is not None:
            graphs.prime(k0, stream)
            for k in range(n):
                graphs.replay(k0 + k)
            return
        if not args.pipeline:
            for k in range(n):
                one_step(k0 + k, timed_dom[k] if timed_dom else None)
            return
        after = None
        if args.text_embed:  # text rows of the packed LLM input, gathered after the return
            def after(k, p, s):
                path.embed_text(p, text_tokens[(k0 + k) % n_distinct], text_table, s)
        path.run_pipeline([(dtabs[(k0 + k) % n_distinct], arenas[(k0 + k) % n_distinct])
                           for k in range(n)], kernel_events=timed_dom, start_event=start_ev,
                          stream=stream, after_step=after)

    graphs = None
    if args.graphs and args.pipeline:
        if n_distinct % 2:
            n_distinct -= 1 if n_distinct > 1 else -1
        graphs = path.capture_steps([dtabs[i % len(dtabs)] for i in range(n_distinct)],
                                    [arenas[i % len(arenas)] for i in range(n_distinct)])
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = Clocks(local)
    with clk:
        t0.record(stream)
        run_steps(0, args.warmup, start_ev=t0)
        t1.record(stream)
        torch.cuda.synchronize()
        # untimed soak (~100 ms) so the clock record covers a loaded GPU
        est = max(t0.elapsed_time(t1) / max(args.warmup, 1), 0.01)
        soak_ms = float(os.environ.get("MUX_BENCH_SOAK_MS", "100"))
        n_soak = torch.tensor([int(min(soak_ms / est, 5000))], device=dev)
        if world > 1:  # every rank must run the same number of exchanges
            dist.all_reduce(n_soak, op=dist.ReduceOp.MIN)
        run_steps(0, int(n_soak.item()))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/
        h0 = time.perf_counter()
        run_steps(args.warmup, args.steps, ev_dom, start_ev=t0)
        path.finish(stream)
        torch.cuda.nvtx.range_pop()
        t1.record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3  # enqueue time: < GPU time = not host-bound
        torch.cuda.synchronize()
    path.check_wait()
    ms = t0.elapsed_time(t1)

    def max_over_ranks(x):
        if world == 1:
            return float(x)
        tt = torch.tensor([float(x)], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    ms = max_over_ranks(ms)
    if world > 1:
        dist.barrier()

    # per-stage breakdown (separate untimed pass, CUDA events between stages)
    # (+ the gradient return of SURVEY §8f-1: dY at the placeholders back to the
    # encoder ranks — measured here, not part of the headline step)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    dy = torch.randn(path.max_llm_rows, d_llm, device=dev).to(torch.bfloat16)
    if not path.staged:  # allocate the gradient windows (collective) and warm up
        path.grad_return(path.plan(dtabs[0], stream), dy, stream)
        torch.cuda.synchronize()
    for k in range(args.steps):
        i = (args.warmup + k) % n_distinct
        ev[k][0].record(stream)
        p = path.plan(dtabs[i], stream)
        ev[k][1].record(stream)
        path.dispatch(p, arenas[i], stream)
        ev[k][2].record(stream)
        path.return_scatter(p, stream)
        ev[k][3].record(stream)
        if not path.staged:  # gradient path is defined for final-row layouts
            path.grad_return(p, dy, stream)
        ev[k][4].record(stream)
    torch.cuda.synchronize()
    path.check_wait()
    stages = {nm: float(np.mean([e[j].elapsed_time(e[j + 1]) for e in ev]))
              for j, nm in enumerate(("plan_ms", "pack_dispatch_ms",
                                      "projector_scatter_ms" if projector else "return_scatter_ms",
                                      "grad_return_ms"))}
    backward = None
    if projector and not path.staged:  # projector backward, after grad_return
        backward = projector_backward_stage(path, dtabs, steps_idx_of(args, n_distinct),
                                            plans_info, dy, stream, ctx)
    # dominant kernel = the return kernel (return+scatter copy, or the projector
    # GEMM), CUDA events on its stream around the launch, over the timed steps
    dom_ms = [a.elapsed_time(b) for a, b in ev_dom] if not graphs else \
        [e[2].elapsed_time(e[3]) for e in ev]

    steps_idx = [(args.warmup + k) % n_distinct for k in range(args.steps)]
    M_total = sum(plans_info[i]["M"] for i in steps_idx)
    T_total = sum(plans_info[i]["T"] for i in steps_idx)
    value = M_total / (ms / 1e3)
    clocks = clk.summary() if rank == 0 else None
    if world > 1:  # every rank picks the same denominator: rank 0's clock record
        obj = [clocks]
        dist.broadcast_object_list(obj, src=0)
        clocks = obj[0]

    # dominant kernel roofline (rank-local)
    hbm, _, _, src = peaks()
    dom_avg_s = float(np.mean(dom_ms)) / 1e3
    my_recv = [sum(plans_info[i]["recv"][g] for i in steps_idx) / len(steps_idx) for g in (0, 1)]
    if projector:
        from paper_2605_08962_b200 import costs
        tf_peak, peak_why = choose_tensor_peak(clocks)
        flops = sum(costs.projector_flops(my_recv[g], d_enc[g], d_llm) for g in (0, 1))
        algo_bytes = sum(my_recv[g] * 2 * (d_enc[g] + d_llm) + 2 * d_enc[g] * d_llm
                         for g in (0, 1) if my_recv[g] > 0)
        roof = {"kernel": "proj_scatter_gemm (tcgen05)", "bound": "tensor",
                "achieved": flops / dom_avg_s / 1e12, "peak": tf_peak, "unit": "TFLOP/s",
                "peak_source": peak_why, "flops_per_launch": flops}
    else:
        ret = sum(plans_info[i]["ret_bytes"] for i in steps_idx) / len(steps_idx)
        algo = 2 * ret  # read + write of every returned row
        algo_bytes = algo
        roof = {"kernel": "segcopy return+scatter", "bound": "hbm",
                "achieved": algo / dom_avg_s / 1e9, "peak": hbm, "unit": "GB/s",
                "peak_source": f"hbm_gbs ({src}); nominal 8000 GB/s",
                "frac_of_nominal_8000": algo / dom_avg_s / 1e9 / 8000.0}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["algorithmic_bytes"] = algo_bytes
    roof["traffic"], roof["traffic_source"] = captured_traffic(name)
    roof["dominant_ms"] = dom_avg_s * 1e3
    if world > 1:
        roof["nvlink"] = nvlink_roofline(path, plans_info, steps_idx, dom_avg_s,
                                         stages["pack_dispatch_ms"], ctx, projector)
        roof["nvlink"]["hardware_counters"] = (
            "none: ncu is single-GPU only and NVML's NVLink byte counters (fields 138-141, "
            "202, 204) answer NOT_SUPPORTED on this pool (scripts/nvml_probe.py)")
    if world > 1 and not projector:  # the exchange is the bottleneck: NVLink is the bound
        roof["hbm_side"] = {k: roof[k] for k in ("bound", "achieved", "peak", "unit", "frac")}
        nv = roof["nvlink"]
        roof.update(bound="nvlink", achieved=nv["return"]["gbs"], peak=nv["peak_gbs"],
                    unit="GB/s", frac=nv["return"]["frac_of_peak"],
                    peak_source=nv["peak_source"])
        cb = nv["return"].get("combined_bound")
        if cb:  # the same kernel against HBM and NVLink together (perfect overlap)
            roof["frac_combined_hbm_nvlink"] = cb["frac"]

    # e2e: public API from pinned host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, path, tables, arenas, plans_info, n_distinct, projector, dev, world)

    # per step: fused planner (1) + dispatch copy (1, + flag wait at N>1) + return:
    # projector: row map (side stream) + one grouped GEMM with the signal fused
    # (+ flag wait at N>1); otherwise one return copy (+ flag wait at N>1);
    # overlapped dispatch at N>1: + consumed signal + its wait
    launches = 1 + 1 + (1 if world > 1 else 0)
    if projector:
        launches += 2 + (1 if world > 1 else 0)
    else:
        launches += 1 + (1 if world > 1 else 0)
    if args.pipeline >= 2 and world > 1:  # consumed wait (+ its signal unless fused in the GEMM)
        launches += 1 if (projector and not path.staged) else 2
    if args.text_embed:
        launches += 1
    line = {
        "metric": "multimodal tokens/s rebalanced+dispatched+scattered per step",
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (reference generator restated; bf16 N(0,1) payload; encoder stand-in)",
        "config": config_dict(name, world, n_distinct, M_total / args.steps,
                              T_total / args.steps),
        "impl_config": {
            "planner": ("pipelined on a side stream" if args.pipeline else "in-line") +
                       ("; dispatch of step k+1 under step k's return"
                        if args.pipeline >= 2 else ""),
            "balance": args.method,
            "lssp": ({"eta": args.lssp_eta, "group": args.lssp_sp or world}
                     if args.lssp_eta >= 0 else None),
            "reshard": args.reshard if sp > 1 else None,
            "text_rows": bool(args.text_embed),
            "launch": "one CUDA graph per step" if graphs is not None else "eager"},
        "roofline": roof,
        "exchange": exchange_summary(plans_info, steps_idx, rank),
        "balance": balance_summary(plans_info, steps_idx),
        "stages": stages,
        "backward": backward,
        "gpu_launches": launches * args.steps,
        "host_enqueue_ms_per_step": host_ms / args.steps,
        "e2e": e2e,
    }
    if projector and world == 1 and not args.no_comparator:
        line["comparator"] = library_comparator(path, dtabs, steps_idx, dom_avg_s * 1e3, stream)
    if rank == 0:
        line["clocks"] = clocks
        if world == 1:
            line["cpu_baseline"] = cpu_baseline(name, tables[0], projector, world, args.method)
    return line


def steps_idx_of(args, n_distinct):
    return [(args.warmup + k) % n_distinct for k in range(args.steps)]


def projector_backward_stage(path, dtabs, steps_idx, plans_info, dy, stream, ctx):
    """dX = G W, dW = G^T X, db (csrc/proj_bwd.cu) of every encoder group after
    each step's gradient return, timed with CUDA events (its own pass, not in
    the headline step); roofline: 4 M d_enc d_llm FLOPs per group."""
    import torch

    from paper_2605_08962_b200 import _lib
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in steps_idx]
    groups = [g for g in range(2) if path.weight[g] is not None]
    for k, i in enumerate([steps_idx[0]] + list(steps_idx)):  # one warm-up step
        p = path.plan(dtabs[i], stream)
        path.grad_return(p, dy, stream)
        a = ev[k - 1] if k else None
        if a:
            a[0].record(stream)
        for g in groups:
            if plans_info[i]["recv"][g]:
                path.projector_backward(g, plan=p, stream=stream)
        if a:
            a[1].record(stream)
    torch.cuda.synchronize()
    path.check_wait()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    flops = np.mean([sum(4.0 * plans_info[i]["recv"][g] * path.d_enc[g] * path.d_llm
                         for g in groups) for i in steps_idx])
    peak, why = choose_tensor_peak(None)
    _, burst, _, _ = peaks()
    return {"ms": ms, "tflops": flops / (ms / 1e3) / 1e12, "peak": burst,
            "frac": flops / (ms / 1e3) / 1e12 / burst,
            "what": "dX = G W (pair GEMM, W^T) + dW = G^T X (pair GEMM, MN-major) + db per "
                    "encoder group, after the gradient return (not timed here); frac of the "
                    "burst bf16 peak",
            "rank": ctx["rank"]}


def combined_bound(per_step, hbm_gbs, link_gbs, t_ms):
    """Roofline of an exchange copy that moves local rows through HBM while it
    pushes remote rows over NVLink.  per_step: [step, sender, receiver] bytes.
    Per rank: HBM bytes = local read + write + egress read + ingress write at
    hbm_gbs; NVLink bytes = max(egress, ingress) at link_gbs.  A step's bound is
    the slower of the two (perfect overlap) on its slowest rank; the bound is the
    mean over the steps (the binding rank and term change from step to step),
    and frac = bound / t_ms (the measured mean exchange time)."""
    bounds, nv_bound = [], 0
    for M in np.asarray(per_step, dtype=np.float64):
        o = M - np.diag(np.diag(M))
        e, i = o.sum(1), o.sum(0)
        t_h = (2 * np.diag(M) + e + i) / (hbm_gbs * 1e9) * 1e3
        t_l = np.maximum(e, i) / (link_gbs * 1e9) * 1e3
        bounds.append(float(np.max(np.maximum(t_h, t_l))))
        nv_bound += int(t_l.max() >= t_h.max())
    bound = float(np.mean(bounds)) if bounds else 0.0
    return {"bound_ms": bound, "frac": bound / t_ms if t_ms > 0 else None,
            "bound_ms_per_step": bounds, "steps_nvlink_bound": nv_bound,
            "hbm_gbs": hbm_gbs, "nvlink_gbs": link_gbs,
            "model": "per timed step: max over ranks of max(HBM bytes / measured HBM, "
                     "NVLink bytes / measured all-to-all push); bound = mean over steps; "
                     "frac = bound / exchange_ms"}


def nvlink_roofline(path, plans_info, steps_idx, ret_s, disp_ms, ctx, projector):
    """Per-GPU NVLink bandwidth of the two exchanges at N > 1.

    Bytes: each rank's return (and dispatch) bytes per destination rank from
    its plan, averaged over the timed steps and all-gathered into the world's
    byte matrix; per rank egress = row sum off the diagonal, ingress = column
    sum.  Time: the exchange kernel's CUDA-event duration, max over ranks.
    Achieved = max over ranks of max(egress, ingress) / that time, the per-GPU
    roofline of SURVEY §8(d).  Peaks measured in this run on the same windows:
    a ring push by the same copy engine (SM stores to the next rank) and the
    copy engine (cudaMemcpyAsync to the peer); NCCL all_to_all_single on the
    same byte matrix is the library comparator."""
    import torch
    import torch.distributed as dist

    world, rank, dev = ctx["world"], ctx["rank"], ctx["dev"]
    n = len(steps_idx)
    mine_ret = sum(plans_info[i]["ret_to"] for i in steps_idx) / n
    mine_disp = sum(plans_info[i]["disp_to"] for i in steps_idx) / n

    def gather(vec):
        t = torch.tensor(vec, dtype=torch.float64, device=dev)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return np.stack([o.cpu().numpy() for o in out])

    def gmax(x):
        t = torch.tensor([float(x)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    Rm, Dm = gather(mine_ret), gather(mine_disp)
    # per-step byte matrices [step, sender, receiver] for the combined bound
    R_steps = gather(np.stack([plans_info[i]["ret_to"] for i in steps_idx])).transpose(1, 0, 2)
    ret_ms, disp_ms = gmax(ret_s * 1e3), gmax(disp_ms)
    probe = nvlink_probe(path, ctx)

    def rec(Mx, t_ms, per_step=None):
        off = Mx - np.diag(np.diag(Mx))
        eg, ing = off.sum(1), off.sum(0)
        b = float(max(eg.max(), ing.max()))
        gbs = b / (t_ms / 1e3) / 1e9 if t_ms > 0 else 0.0
        r = {"remote_bytes_max_rank": b, "egress_bytes": eg.tolist(),
             "ingress_bytes": ing.tolist(), "local_bytes": np.diag(Mx).tolist(),
             "exchange_ms": t_ms, "gbs": gbs, "frac_of_peak": gbs / probe["peak_gbs"],
             "frac_of_alltoall": gbs / probe["alltoall_gbs"] if probe.get("alltoall_gbs")
             else None,
             "frac_of_900": gbs / 900.0}
        if per_step is not None and t_ms > 0:
            r["combined_bound"] = combined_bound(per_step, peaks()[0],
                                                 probe.get("alltoall_gbs") or probe["peak_gbs"],
                                                 t_ms)
        return r

    out = {"return": rec(Rm, ret_ms, per_step=None if projector else R_steps),
           "dispatch": rec(Dm, disp_ms),
           "peak_gbs": probe["peak_gbs"],
           "peak_source": probe["peak_source"],
           "probe": probe,
           "nominal_gbs": 900.0,
           "note": "return: the kernel timed in the step loop (projector: the GEMM whose "
                   "epilogue stores remote rows); dispatch: the pack+dispatch stage of the "
                   "in-line stage pass (includes its flag wait)"}
    out["nccl_all_to_allv"] = nccl_comparator(Rm, ctx)
    out["return"]["vs_nccl"] = out["nccl_all_to_allv"]["ms"] / ret_ms if ret_ms else None
    return out


def nvlink_probe(path, ctx, nbytes=256 << 20, iters=5):
    """Ring push of `nbytes` from every rank to rank+1's receive window: SM
    stores (mux_copy_bytes, the exchange's copy engine) and the copy engine
    (cudaMemcpyAsync to the peer pointer).  Max over ranks of CUDA-event time."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2605_08962_b200 import _lib
    world, rank, dev = ctx["world"], ctx["rank"], ctx["dev"]
    win = path.recv[0]
    nbytes = min(nbytes, win.tensor.numel()) & ~((1 << 20) - 1)
    if nbytes == 0:  # a window too small to probe: fall back to the nominal figure
        return {"bytes": 0, "peak_gbs": 900.0, "alltoall_gbs": None,
                "peak_source": "nominal (window too small to probe)"}
    src = torch.empty(nbytes, dtype=torch.uint8, device=dev).fill_(rank)
    dst = win.ptrs[(rank + 1) % world]
    L = _lib.lib()
    s = torch.cuda.current_stream()
    # all-to-all: nbytes split over every peer, written concurrently by one launch,
    # each source rank into its own slice of every peer's window
    share = (min(nbytes // max(world - 1, 1), win.tensor.numel() // world)) & ~4095
    peers = [r for r in range(world) if r != rank]
    a2a = [torch.tensor(v, dtype=torch.int64, device=dev) for v in (
        [win.ptrs[r] + rank * share for r in peers],
        [src.data_ptr() + k * share for k in range(len(peers))], [share] * len(peers))]
    res = {}
    for nm, fn, moved in (
            ("sm_push_ring", lambda: L.mux_copy_bytes(C.c_void_p(dst), C.c_void_p(src.data_ptr()),
                                                      nbytes, 0, C.c_void_p(s.cuda_stream)),
             nbytes),
            ("copy_engine_ring", lambda: L.mux_memcpy_async(C.c_void_p(dst),
                                                            C.c_void_p(src.data_ptr()), nbytes,
                                                            C.c_void_p(s.cuda_stream)), nbytes),
            ("sm_push_alltoall", lambda: L.mux_copy_ranges(
                len(peers), a2a[0].data_ptr(), a2a[1].data_ptr(), a2a[2].data_ptr(), share, 0, 0,
                C.c_void_p(s.cuda_stream)), share * len(peers))):
        _lib.check(fn(), nm)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(iters):
            _lib.check(fn(), nm)
        b.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[nm + "_gbs"] = moved / (float(t.item()) / 1e3) / 1e9
        dist.barrier()
    res["bytes"] = nbytes
    res["peak_gbs"] = max(res["sm_push_ring_gbs"], res["copy_engine_ring_gbs"])
    res["peak_source"] = ("measured in this run: best of SM-store ring push and copy-engine "
                          "ring push, 1 peer per rank, per direction")
    res["alltoall_gbs"] = res["sm_push_alltoall_gbs"]
    return res


def nccl_comparator(Mx, ctx, iters=5):
    """NCCL all_to_all_single with the exchange's byte matrix (row = sender,
    column = receiver; the diagonal is the local part, as in our kernel)."""
    import torch
    import torch.distributed as dist

    world, rank, dev = ctx["world"], ctx["rank"], ctx["dev"]
    sizes = np.rint(Mx).astype(np.int64)
    send = [int(x) for x in sizes[rank]]
    recv = [int(sizes[s, rank]) for s in range(world)]
    inp = torch.empty(max(sum(send), 1), dtype=torch.uint8, device=dev)
    out = torch.empty(max(sum(recv), 1), dtype=torch.uint8, device=dev)
    if sum(send) == 0 and sum(recv) == 0:
        return {"ms": 0.0}
    for _ in range(2):
        dist.all_to_all_single(out[:sum(recv)], inp[:sum(send)], recv, send)
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(iters):
        dist.all_to_all_single(out[:sum(recv)], inp[:sum(send)], recv, send)
    b.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / iters], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    off = sizes - np.diag(np.diag(sizes))
    b_max = float(max(off.sum(1).max(), off.sum(0).max()))
    return {"ms": ms, "gbs": b_max / (ms / 1e3) / 1e9 if ms > 0 else 0.0,
            "what": "torch.distributed.all_to_all_single (NCCL) of the same per-rank byte "
                    "matrix into contiguous buffers, max over ranks"}


def library_comparator(path, dtabs, steps_idx, fused_ms, stream, reps=None):
    """Same-shape library path for the fused projector + scatter: cuBLAS
    (torch.matmul) into a temporary, + bias, then index_copy_ of the rows into
    the packed LLM buffer, on the same steps' encoder rows and row maps."""
    import torch

    from paper_2605_08962_b200 import _lib
    reps = reps or len(steps_idx)
    jobs = []
    for i in sorted(set(steps_idx)):
        p = path.plan(dtabs[i], stream)
        h = p.header()
        rmap = torch.empty_like(path.row_dst)
        path._row_map(p, rmap, stream)
        for g in range(2):
            m = int(h[_lib.H_RECV_ROWS0 + g])
            if m and path.weight[g] is not None:
                idx = (rmap[g * path.max_rows: g * path.max_rows + m] & ((1 << 40) - 1))
                jobs.append((i, g, m, idx))
    torch.cuda.synchronize()
    llm = path.llm_view()
    by_step = {}
    for (i, g, m, idx) in jobs:
        by_step.setdefault(i, []).append((g, m, idx))

    def one(i):
        for (g, m, idx) in by_step.get(i, []):
            x = path.enc_view(g, m)
            y = torch.addmm(path.bias[g], x, path.weight[g].t())
            llm.index_copy_(0, idx, y)

    ys = {(i, g): torch.empty(m, path.d_llm, dtype=torch.bfloat16, device=llm.device)
          for i, jobs_i in by_step.items() for (g, m, _) in jobs_i}

    def gemm_only(i):  # the same GEMMs into preallocated outputs, no scatter
        for (g, m, idx) in by_step.get(i, []):
            torch.addmm(path.bias[g], path.enc_view(g, m), path.weight[g].t(), out=ys[(i, g)])

    def timed(fn):
        for i in sorted(set(steps_idx)):  # warm every step's shapes (cuBLAS heuristics)
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(reps):
            fn(steps_idx[k % len(steps_idx)])
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    lib_ms = timed(one)
    gemm_ms = timed(gemm_only)
    rows = np.mean([sum(m for (g, m, _) in by_step.get(i, [])) for i in steps_idx])
    flops = 2.0 * rows * path.d_enc[0] * path.d_llm
    return {"library": "torch.addmm (cuBLAS, bf16) + index_copy_ into the packed LLM rows",
            "library_ms": lib_ms, "fused_ms": fused_ms, "speedup": lib_ms / fused_ms,
            "cublas_gemm_only_ms": gemm_ms,
            "cublas_gemm_only_tflops": flops / (gemm_ms / 1e3) / 1e12,
            "fused_tflops": flops / (fused_ms / 1e3) / 1e12,
            "note": "cublas_gemm_only: the same-shape GEMM alone (no scatter, no bias-free "
                    "shortcut) — the library's throughput at this M x 1280 x 4096 shape"}


def captured_traffic(name):
    """DRAM bytes (read + write) of one launch of the dominant kernel from an
    `ncu --set full` capture (profiles/traffic.json), or (None, why).  The
    captured launch's own algorithmic bytes are named in the source string:
    compare ratios, since the captured step may differ from the timed mix."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            rec = json.load(f).get(name)
    except (OSError, ValueError):
        rec = None
    if not rec:
        return None, f"no ncu capture for {name} in profiles/traffic.json"
    t = rec["dram_read"] + rec["dram_write"]
    return t, (f"ncu --set full of one launch ({rec['summary']}; {rec['launch']}): dram r+w "
               f"{t} B vs that launch's algorithmic {rec['algorithmic_bytes']} B "
               f"(ratio {t / rec['algorithmic_bytes']:.3f})")


def run_e2e(args, path, tables, arenas, plans_info, n_distinct, projector, dev, world):
    """e2e, both loader transfers; the faster is the headline (see run_e2e_one)."""
    a = run_e2e_one(args, path, tables, arenas, plans_info, n_distinct, projector, dev, world,
                    fused_loader=False)
    b = run_e2e_one(args, path, tables, arenas, plans_info, n_distinct, projector, dev, world,
                    fused_loader=True)
    best = dict(a if a["value"] >= b["value"] else b)
    best["variants"] = {"copy_engine_upload": {k: a[k] for k in ("value", "ms_per_step")},
                        "fused_loader": {k: b[k] for k in ("value", "ms_per_step")}}
    return best


def run_e2e_one(args, path, tables, arenas, plans_info, n_distinct, projector, dev, world,
                fused_loader=False):
    """The same steps through the public API from pinned host memory.

    Every step moves its step table and loader payload host->device and reads
    its plan header back (D2H), inside the timed region.  Like a data loader
    with pinned memory, the upload of step k+1 runs on a copy stream
    (MuxPath.run_pipeline's `prepare`) and its plan on the planner stream while
    step k's rows move, with the same overlapped dispatch as `value`; two device
    input slots alternate.  fused_loader=True: only the step
    table is uploaded; the dispatch kernel reads the loader rows straight from
    pinned host memory (UVA) into the encoder ranks' receive windows, so the
    payload crosses PCIe once and is never staged in HBM."""
    import torch
    import torch.distributed as dist

    from paper_2605_08962_b200 import _lib
    from paper_2605_08962_b200.planner import DeviceTable

    host_tabs = [torch.from_numpy(t.blob()).pin_memory() for t in tables]
    host_ar = [[a.cpu().pin_memory() for a in ar] for ar in arenas]
    width = [max(ar[g].numel() for ar in arenas) for g in range(2)]
    dev_ar = [[torch.empty(width[g], dtype=torch.bfloat16, device=dev) for g in range(2)]
              for _ in range(2)]
    dev_tab = [torch.empty(max(h.numel() for h in host_tabs), dtype=torch.int64, device=dev)
               for _ in range(2)]
    out_hdr = [torch.empty(_lib.H_SLOTS, dtype=torch.int64).pin_memory() for _ in range(2)]
    stream = torch.cuda.current_stream()
    up = torch.cuda.Stream(dev)
    uploaded = [torch.cuda.Event() for _ in range(2)]
    consumed = [None, None]
    steps = max(args.steps, 3)
    trace = None  # MUX_E2E_TRACE=1: per-step upload / step-end events to stderr
    counts = {"h2d": 0, "d2h": 0}

    def mark(name, k, s):
        if trace is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            trace.append((name, k, e, time.perf_counter()))

    def prepare(k):
        """Upload step k into input slot k % 2 (the loader side of the pipeline)."""
        i, slot = k % n_distinct, k % 2
        if consumed[slot] is not None:  # step k-2 is done with this slot
            up.wait_event(consumed[slot])
        mark("up", k, up)
        with torch.cuda.stream(up):
            blob = dev_tab[slot][: host_tabs[i].numel()]
            blob.copy_(host_tabs[i], non_blocking=True)
            mark("tab", k, up)
            if not fused_loader:
                for g in range(2):
                    n = host_ar[i][g].numel()
                    dev_ar[slot][g][:n].copy_(host_ar[i][g].view(-1), non_blocking=True)
        uploaded[slot].record(up)
        mark("up_end", k, up)
        counts["h2d"] += host_tabs[i].numel() * 8 + sum(b.numel() * 2 for b in host_ar[i])
        if fused_loader:  # the dispatch kernel reads the pinned rows over PCIe
            shaped = host_ar[i]
        else:
            shaped = [dev_ar[slot][g][: host_ar[i][g].numel()].view(host_ar[i][g].shape)
                      for g in range(2)]
        return DeviceTable.from_blob(tables[i], blob), shaped, uploaded[slot]

    def after(k, p, s):
        """Read the step's plan header back (D2H) and release its input slot once
        every reader of the step's inputs ran (path.step_done: the event after
        which the step's plan and inputs are no longer read)."""
        slot = k % 2
        if path.step_done is not None:
            s.wait_event(path.step_done)
        out_hdr[slot].copy_(p.view("header", _lib.H_SLOTS), non_blocking=True)
        mark("step_end", k, s)
        c = torch.cuda.Event()
        c.record(s)
        consumed[slot] = c
        counts["d2h"] += 8 * _lib.H_SLOTS

    def run(n):
        path.run_pipeline(n=n, prepare=prepare, after_step=after, stream=stream)

    # warm-up over every distinct step: each pinned host buffer is DMA'd once
    # before timing (a first DMA from freshly pinned pages runs at 23-40 of the
    # 55 GB/s, scripts/probes/pinned_upload_probe.py; a loader reuses its pinned
    # staging buffers, so the steady state is what the timed steps measure)
    run(max(3, n_distinct))
    torch.cuda.synchronize()
    path.check_wait()
    if world > 1:
        dist.barrier()
    counts.update(h2d=0, d2h=0)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if os.environ.get("MUX_E2E_TRACE"):
        trace = []
    t0.record(stream)
    th0 = time.perf_counter()
    up.wait_event(t0)
    run(steps)
    path.finish(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    path.check_wait()
    ms = t0.elapsed_time(t1)
    if trace:
        print("e2e trace (fused_loader=%s, gpu ms / host-enqueue ms):" % fused_loader, " ".join(
            f"{n}{k}@{t0.elapsed_time(e):.3f}/{(h - th0) * 1e3:.3f}" for n, k, e, h in trace),
            file=sys.stderr)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    assert all(int(h[_lib.H_STATUS]) == 0 for h in out_hdr)
    M = sum(plans_info[k % n_distinct]["M"] for k in range(steps))
    return {"value": M / (ms / 1e3), "unit": "tokens/s",
            "h2d_bytes_per_step": counts["h2d"] // steps,
            "d2h_bytes_per_step": counts["d2h"] // steps, "steps": steps, "ms_per_step": ms / steps,
            "loader": "fused: dispatch kernel reads pinned host rows (UVA)" if fused_loader else
                      "copy engine upload to a device slot, then the dispatch copy",
            "note": "per step: step table + loader payload host->device from pinned host memory "
                    "(one step ahead) and the plan header D2H, all inside the window"}


# ----------------------------------------------------------------------------
# CPU reference arm (the reference's own packer + the oracle port of the
# SPEC-only balance/reshard and of the data plane; the reference itself never
# moves token data)
# ----------------------------------------------------------------------------

def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _reference_workload():
    """The reference's own muxsim.workload from baseline/_ref (installed from
    /root/reference/pkg), or None when it is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "muxsim")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import muxsim.workload as RW
        return RW
    except Exception:
        return None


def reference_pack(RW, table, capacity):
    """The reference's hybrid_pack on every drawn chunk of the step table (its
    own code, workload.py:240-262) after the carried sequences, then its
    build_global_batch is left to the caller.  Returns (sequences, seconds)
    with only the hybrid_pack calls inside the timing."""
    mods = {0: "text", 1: "image", 2: "video", 3: "audio"}
    lens, ids, tmods = table["lens"], table["ids"], table["mods"]
    nc = len(table["carry_seq"])
    seqs = [RW.PackedSequence(capacity=capacity) for _ in range(int(table["n_carry_seqs"]))]
    for i in range(nc):
        seqs[int(table["carry_seq"][i])].spans.append((int(ids[i]), int(lens[i])))
    chunks = []
    co = list(table["chunk_off"])
    for c in range(len(co) - 1):
        chunks.append([RW.Sample(int(ids[i]), RW.Modality(mods[int(tmods[i])]), "synthetic",
                                 int(lens[i])) for i in range(co[c], co[c + 1])])
    t0 = time.perf_counter()
    for ch in chunks:
        seqs.extend(RW.hybrid_pack(ch, capacity))
    return seqs, time.perf_counter() - t0


def cpu_baseline(name, table, projector, world=1, method="lpt_local", weights=None):
    """Time the CPU path on one step of the workload at `world` GPUs' scale.

    Code timed: the reference's own hybrid_pack + build_global_batch from
    baseline/_ref (workload.py:240-278; the oracle restatement when that is
    absent), the oracle port of the SPEC-only balance / reshard / segment
    tables, and the data plane in torch-CPU over all ranks' rows at once
    (index_select pack, index_copy_ return/scatter, and the projector as an
    fp32-accumulate matmul over every row).  All host threads.  One step = the
    bounded sample."""
    import torch

    from oracle import planner as oplan
    from paper_2605_08962_b200 import configs

    cfg, dp, sp, gbs = workload(name, world)
    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    t = dict(lens=table.lens.astype(np.int64), mods=table.mods.astype(np.int64), ids=table.ids,
             carry_seq=table.carry_seq.astype(np.int64), n_carry_seqs=table.n_carry_seqs,
             chunk_off=table.chunk_off.tolist())
    d_in, d_enc, d_llm = configs.D_IN, configs.D_ENC, configs.D_LLM
    RW = _reference_workload()
    if RW is not None:
        seqs, t_pack_ref = reference_pack(RW, t, configs.CAPACITY)
        t0 = time.perf_counter()
        RW.build_global_batch(seqs, 0, gbs, dp, 1)
        packed = oplan.packed_from_sequences(t, seqs)
        o = oplan.plan_step(t, configs.CAPACITY, gbs, dp, sp, world, 1, method, packed=packed)
        t_plan = t_pack_ref + time.perf_counter() - t0
        planner_kind = ("reference hybrid_pack + build_global_batch (baseline/_ref) + oracle "
                        "balance/reshard/segments")
    else:
        t0 = time.perf_counter()
        o = oplan.plan_step(t, configs.CAPACITY, gbs, dp, sp, world, 1, method)
        t_plan = time.perf_counter() - t0
        planner_kind = "oracle planner (baseline/_ref absent)"
    lens = t["lens"]
    items = np.flatnonzero(o["enc"] >= 0)
    rows = [int(o["arena_rows"][:, g].sum()) for g in range(2)]
    # all ranks' arenas / receive buffers / LLM buffers stacked: one global row space
    a_base = np.zeros((world, 2), np.int64)
    r_base = np.zeros((world, 2), np.int64)
    for g in range(2):
        a_base[1:, g] = np.cumsum(o["arena_rows"][:-1, g])
        r_base[1:, g] = np.cumsum(o["recv_rows"][:-1, g])
    l_base = np.zeros(world, np.int64)
    l_base[1:] = np.cumsum(o["llm_rows"][:-1])
    arenas = [torch.randn(max(r, 1), d_in[g]).to(torch.bfloat16) for g, r in enumerate(rows)]
    recv = [torch.empty(max(r, 1), d_in[g], dtype=torch.bfloat16) for g, r in enumerate(rows)]
    d_ret = d_enc if projector else (d_llm, d_llm)
    enc = [torch.randn(max(r, 1), d_ret[g]).to(torch.bfloat16) for g, r in enumerate(rows)]
    Ws = [torch.randn(d_llm, d_enc[g]).to(torch.bfloat16) for g in range(2)] if projector \
        else None
    llm = torch.zeros(int(o["llm_rows"].sum()), d_llm, dtype=torch.bfloat16)
    t0 = time.perf_counter()
    for g in range(2):  # pack + dispatch: origin arena rows -> encoder receive rows
        src, dst = [], []
        for i in items:
            if o["group"][i] == g:
                L = int(lens[i])
                a = a_base[o["origin"][i], g] + o["arena_off"][i]
                r = r_base[o["enc"][i], g] + o["enc_off"][i]
                src.append(np.arange(a, a + L))
                dst.append(np.arange(r, r + L))
        if src:
            sI, dI = torch.from_numpy(np.concatenate(src)), torch.from_numpy(np.concatenate(dst))
            recv[g].index_copy_(0, dI, arenas[g].index_select(0, sI))
    t_pack = time.perf_counter() - t0
    t0 = time.perf_counter()
    for g in range(2):  # return (+ projector) + scatter into the packed LLM rows
        src, dst = [], []
        for (i, sr, dr_rank, dr, n) in o["pieces"]:
            if o["group"][i] == g:
                e = r_base[o["enc"][i], g]
                src.append(np.arange(e + sr, e + sr + n))
                dst.append(np.arange(l_base[dr_rank] + dr, l_base[dr_rank] + dr + n))
        if not src:
            continue
        sI, dI = torch.from_numpy(np.concatenate(src)), torch.from_numpy(np.concatenate(dst))
        x = enc[g].index_select(0, sI)
        if projector:  # every row, fp32 accumulate, rounded to bf16
            x = (x.float() @ Ws[g].float().t()).to(torch.bfloat16)
        llm.index_copy_(0, dI, x)
    t_ret = time.perf_counter() - t0
    M = int(o["recv_rows"].sum())
    total = t_plan + t_pack + t_ret
    sample = (f"one {name} step at {world} GPU(s) simulated in-process: {M} modality tokens; "
              f"{planner_kind}; torch-CPU gather/scatter"
              + ("; fp32 projector over all rows" if projector else ""))
    return {"value": M / total, "unit": "tokens/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "sample": sample,
            "seconds": {"plan": t_plan, "pack": t_pack, "return": t_ret},
            "step_seconds": total, "M": M, "T": int(o["llm_rows"].sum())}


def run_reference(args):
    """CPU reference arm: rank 0 only; the other ranks exit without work.  The
    same distinct steps in the same order as our arm's timed region, and the
    same `config`."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    cfg, dp, sp, gbs = workload(name, world)
    n_distinct = n_distinct_of(args)
    tables = generate_steps_host(name, world, n_distinct)
    vals = []
    for k in range(args.warmup + args.steps):
        r = cpu_baseline(name, tables[k % n_distinct], bool(cfg["projector"]), world,
                         args.method)
        if k >= args.warmup:
            vals.append(r)
    secs = sum(r["step_seconds"] for r in vals)
    M = sum(r["M"] for r in vals)
    v = M / secs
    line = {"metric": "multimodal tokens/s rebalanced+dispatched+scattered per step",
            "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / len(vals) * 1e3,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference generator restated; bf16 N(0,1) payload; encoder stand-in)",
            "impl": "reference",
            "config": config_dict(name, world, n_distinct, M / len(vals),
                                  sum(r["T"] for r in vals) / len(vals)),
            "impl_config": {"ranks": f"{world} simulated in-process on the host",
                            "balance": args.method},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": vals[0]["cores"],
                             "kind": "port", "cpu_model": vals[0]["cpu_model"],
                             "sample": vals[0]["sample"],
                             "seconds_per_step": {k: float(np.mean([r["seconds"][k]
                                                                     for r in vals]))
                                                  for k in ("plan", "pack", "return")}},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def generate_steps_host(name, world, n_steps):
    """Same step tables as generate_steps, produced by the CPU oracle generator."""
    from oracle import planner as oplan
    from oracle import workload as owork
    from paper_2605_08962_b200 import configs
    from paper_2605_08962_b200.planner import StepTable
    cfg, dp, sp, gbs = workload(name, world)
    descs = owork.descs_from_config(configs.DATASETS, cfg["datasets"])
    carry, seen, out = None, {}, []
    for step in range(n_steps):
        b, rest, drawn, chunks = owork.generate(descs, cfg["phases"], False, step, cfg["seed"],
                                                gbs, dp, 1, configs.CAPACITY,
                                                carry if cfg["carry"] else None)
        for smp in drawn:
            seen[smp[0]] = smp[1]
        t = oplan.step_table(list(carry or []) if cfg["carry"] else [], drawn, chunks, seen)
        out.append(StepTable(t["lens"].astype(np.int32), t["mods"].astype(np.int32), t["ids"],
                             t["carry_seq"].astype(np.int32), t["n_carry_seqs"],
                             np.asarray(t["chunk_off"], np.int32)))
        carry = rest
    return out


def main():
    args = parse()
    if args.hang_dump > 0:
        import faulthandler
        faulthandler.dump_traceback_later(args.hang_dump, exit=False)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
