"""Per-rank event timeline of the OVERLAPPED pipeline (MuxPath.run_pipeline, the
bench default): where the main stream's time goes between GEMMs/returns.

    torchrun --nproc-per-node N scripts/ov_timeline.py [config] [steps]
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
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 24
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
                   projector=proj, device=dev, group=group, method="lpt_local",
                   overlap_dispatch=True)
    path.dispatch_grid = -2 * path.num_sms
    if proj:
        for g in range(2):
            path.set_projector(g, (torch.randn(configs.D_LLM, configs.D_ENC[g], device=dev)
                                   / 32).to(torch.bfloat16))
    dtabs = [DeviceTable(t, dev) for t in tables]
    arenas = []
    for d in dtabs:
        pl = path.plan(d)
        path.encode_standin(pl, d)
        info = pl.host()
        arenas.append([torch.randn(max(int(info["arena_rows"][rank, g]), 1), configs.D_IN[g],
                                   device=dev).to(torch.bfloat16) for g in range(2)])
    st = torch.cuda.current_stream()
    seq = [(dtabs[k % 8], arenas[k % 8]) for k in range(steps)]
    marks = {k: {} for k in range(steps)}
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]

    def enc(k, p, s):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        marks[k]["enc"] = e

    def after(k, p, s):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        marks[k]["after"] = e

    path.run_pipeline(seq[:6], stream=st)  # warm
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    path.run_pipeline(seq, encoder=enc, after_step=after, kernel_events=kev, stream=st)
    torch.cuda.synchronize()
    rows = []
    for k in range(3, steps - 1):
        e0 = marks[k]["enc"]
        rows.append({
            "E signal + launch": e0.elapsed_time(kev[k][0]) * 1e3,
            "return kernel": kev[k][0].elapsed_time(kev[k][1]) * 1e3,
            "return wait": kev[k][1].elapsed_time(marks[k]["after"]) * 1e3,
            "to next step": marks[k]["after"].elapsed_time(marks[k + 1]["enc"]) * 1e3,
            "period": e0.elapsed_time(marks[k + 1]["enc"]) * 1e3})
    mean = {kk: round(float(np.mean([r[kk] for r in rows])), 1) for kk in rows[0]}
    print(json.dumps({"rank": rank, "world": world, "config": name, "mean_us": mean}),
          flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
