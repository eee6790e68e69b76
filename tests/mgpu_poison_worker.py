"""torchrun worker: the failure path across GPUs.

    torchrun --nproc-per-node N tests/mgpu_poison_worker.py

Step 0 runs normally.  In step 1 the last rank does not launch its dispatch, so
every other rank's flag wait times out (short timeout), poisons that rank's
path, and the poisoned return copies publish the poison bit — the last rank's
return wait then ends poisoned too (status 2 if the poisoned flags arrive first,
1 if its own timeout fires first).  Every rank must end with a raised
RuntimeError from check_wait(), and a poisoned rank's own return rows stay
unwritten.  Then every rank calls reset_status() and a third step runs healthy
with step 0's results.  Every wait is bounded; no kernel hangs."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import planner as oplan  # noqa: E402
from oracle import workload as owork  # noqa: E402
from paper_2605_08962_b200 import configs, planner  # noqa: E402
from paper_2605_08962_b200.dataplane import MuxPath  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    cfg = configs.CONFIGS["cfg5"]
    gbs = cfg["gbs_per_replica"] * world
    descs = owork.descs_from_config(configs.DATASETS, cfg["datasets"])
    _, _, drawn, chunks = owork.generate(descs, cfg["phases"], False, 0, cfg["seed"], gbs, world,
                                         1, configs.CAPACITY)
    t = oplan.step_table([], drawn, chunks, {})
    o = oplan.plan_step(t, configs.CAPACITY, gbs, world, 1, world)
    d_in, d_llm = (20, 8), 64
    path = MuxPath(capacity=configs.CAPACITY, gbs=gbs, dp=world, world=world, rank=rank,
                   d_in=d_in, d_llm=d_llm, device=dev, group=dist.group.WORLD,
                   wait_timeout_ms=300)
    table = planner.StepTable(t["lens"].astype(np.int32), t["mods"].astype(np.int32), t["ids"],
                              t["carry_seq"].astype(np.int32), 0,
                              np.asarray(t["chunk_off"], np.int32))
    dtab = planner.DeviceTable(table, dev)
    arenas = [torch.randn(max(int(o["arena_rows"][rank, g]), 1), d_in[g], device=dev)
              .to(torch.bfloat16) for g in range(2)]
    ok = True
    plan = path.plan(dtab)
    plan.check(table)
    # step 0: healthy
    path.dispatch(plan, arenas)
    path.encode_standin(plan, dtab)
    path.return_scatter(plan)
    torch.cuda.synchronize()
    path.check_wait()
    step0_llm = path.llm_view(int(o["llm_rows"][rank])).clone()
    dist.barrier()
    # step 1: the last rank skips its dispatch
    path.zero_llm()
    torch.cuda.synchronize()
    dist.barrier()
    if rank != world - 1:
        path.dispatch(plan, arenas)
    path.encode_standin(plan, dtab)
    path.return_scatter(plan)
    torch.cuda.synchronize()
    code = int(path.wait_err.item())
    try:
        path.check_wait()
        ok = False  # must raise
    except RuntimeError as e:
        ok &= "poisoned" in str(e)
    ok &= code in (1, 2)
    if rank != world - 1:
        ok &= code == 1  # its dispatch wait timed out (the last rank never signalled)
    # a poisoned path moves nothing: the rows this rank would have returned into its
    # own LLM buffer stay zero (the last rank, poisoned only later, did copy)
    if rank != world - 1:  # poisoned before its return copy (its dispatch wait timed out)
        n = int(o["llm_rows"][rank])
        llm = path.llm_view(n)
        for (i, src, dst_rank, dst_row, k) in o["pieces"]:
            if int(o["enc"][i]) == rank and dst_rank == rank and k:
                ok &= bool((llm[dst_row:dst_row + k] == 0).all())
    # recovery: every rank resets its status and flags together; the next step is
    # healthy again and its LLM rows match step 0's (same plan, same inputs)
    ref = None
    path.reset_status()
    path.zero_llm()
    torch.cuda.synchronize()
    dist.barrier()
    path.dispatch(plan, arenas)
    path.encode_standin(plan, dtab)
    path.return_scatter(plan)
    torch.cuda.synchronize()
    try:
        path.check_wait()
    except RuntimeError:
        ok = False
    n = int(o["llm_rows"][rank])
    ref = step0_llm
    ok &= torch.equal(path.llm_view(n), ref)
    print(f"rank {rank}: status {code} ok={ok}", flush=True)
    t_ok = torch.tensor([int(ok)], device=dev)
    dist.all_reduce(t_ok, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if int(t_ok.item()) else 1)


if __name__ == "__main__":
    main()
