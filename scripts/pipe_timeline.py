"""Event timeline of the PIPELINED step loop (what bench.py times), per rank.

    torchrun --nproc-per-node N scripts/pipe_timeline.py [config] [steps]

The plan of step k+1 runs on the planner's side stream during step k (as in
bench.py); CUDA events on both streams give, per step, when each stage starts
and ends relative to the step's first event.  No profiler.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08962_b200 import configs  # noqa: E402
from paper_2605_08962_b200.dataplane import MuxPath  # noqa: E402
from paper_2605_08962_b200.planner import DeviceTable  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    cfg, dp, sp, gbs = bench.workload(name, world)
    proj = bool(cfg["projector"])
    tables = bench.generate_steps(name, world, 8)
    path = MuxPath(capacity=configs.CAPACITY, gbs=gbs, dp=dp, sp=sp, world=world, rank=rank,
                   d_in=configs.D_IN, d_enc=configs.D_ENC, d_llm=configs.D_LLM,
                   projector=proj, device=dev, group=group,
                   method=os.environ.get("MUX_METHOD", "lpt_local"))
    if proj:
        for g in range(2):
            path.set_projector(g, torch.randn(configs.D_LLM, configs.D_ENC[g], device=dev)
                               .to(torch.bfloat16))
    dtabs = [DeviceTable(t, dev) for t in tables]
    arenas = []
    for d in dtabs:
        info = path.plan(d).host()
        arenas.append([torch.randn(max(int(info["arena_rows"][rank, g]), 1), configs.D_IN[g],
                                   device=dev).to(torch.bfloat16) for g in range(2)])
    st = torch.cuda.current_stream()
    R = path.RING

    def ev(stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def loop(n, record):
        marks = []
        path.plan_ahead(dtabs[0], 0)
        for k in range(n):
            m = {}
            if k + 1 < n:
                path._ensure_ring()
                m["plan+1 start"] = ev(path._side)
                path.plan_ahead(dtabs[(k + 1) % len(dtabs)], (k + 1) % R)
                m["plan+1 end"] = ev(path._side)
            m["step start"] = ev(st)
            st.wait_event(path._ready[k % R])
            m["plan ready"] = ev(st)
            p = path._ring[k % R]
            path.dispatch(p, arenas[k % len(arenas)], st)
            m["dispatch end"] = ev(st)
            e = path.return_scatter(p, st)
            path._freed[k % R] = e
            m["return end"] = ev(st)
            marks.append(m)
        return marks

    loop(6, False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    marks = loop(steps, True)
    torch.cuda.synchronize()
    rows = []
    for k in range(2, steps - 1):
        m, nxt = marks[k], marks[k + 1]
        t0 = m["step start"]
        r = {key: round(t0.elapsed_time(e) * 1e3, 1) for key, e in m.items()}
        r["next step start"] = round(t0.elapsed_time(nxt["step start"]) * 1e3, 1)
        rows.append(r)
    keys = list(rows[0].keys())
    mean = {kk: round(float(np.mean([r[kk] for r in rows])), 1) for kk in keys}
    print(json.dumps({"rank": rank, "world": world, "config": name, "mean_us": mean}),
          flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
