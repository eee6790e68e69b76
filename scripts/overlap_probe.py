"""Timeline of the pipelined step on both streams (main, comm, side) of every rank.

    torchrun --nproc-per-node N scripts/overlap_probe.py [config] [steps]

Issues the bench's pipelined loop with events around every stage on the stream
it runs on, all measured from one reference event, and prints per-step start /
end microseconds for: plan (side), dispatch (main), GEMM (main), push (comm).
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08962_b200 import configs  # noqa: E402
from paper_2605_08962_b200.dataplane import MuxPath  # noqa: E402
from paper_2605_08962_b200.planner import DeviceTable  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD
    cfg, dp, sp, gbs = bench.workload(name, world)
    proj = bool(cfg["projector"])
    tables = bench.generate_steps(name, world, 4)
    path = MuxPath(capacity=configs.CAPACITY, gbs=gbs, dp=dp, sp=sp, world=world, rank=rank,
                   d_in=configs.D_IN, d_enc=configs.D_ENC, d_llm=configs.D_LLM,
                   projector=proj, device=dev, group=group)
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
    torch.cuda.synchronize()
    main_s = torch.cuda.current_stream()

    def ev(stream):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    for rep in range(2):
        if world > 1:
            dist.barrier()
        ref = ev(main_s)
        rec = []
        R = path.RING
        path.plan_ahead(dtabs[0], 0, after=ref)
        for k in range(steps):
            r = {}
            if k + 1 < steps:
                path._ensure_ring()
                a = ev(path._side)
                path.plan_ahead(dtabs[(k + 1) % len(dtabs)], (k + 1) % R)
                r["plan_next"] = (a, ev(path._side))
            main_s.wait_event(path._ready[k % R])
            a = ev(main_s)
            p = path._ring[k % R]
            path.dispatch(p, arenas[k % len(arenas)], main_s)
            r["dispatch"] = (a, ev(main_s))
            a = ev(main_s)
            done = path.return_scatter(p, main_s)
            r["gemm"] = (a, ev(main_s))
            if done is not None:
                r["push_done"] = (a, done)
            else:
                done = ev(main_s)
            path._freed[k % R] = done
            rec.append(r)
        path.finish(main_s)
        torch.cuda.synchronize()
    out = []
    for k, r in enumerate(rec):
        row = {}
        for nm, (a, b) in r.items():
            row[nm] = [round(ref.elapsed_time(a) * 1e3), round(ref.elapsed_time(b) * 1e3)]
        out.append(row)
    print(json.dumps({"rank": rank, "steps": out}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
