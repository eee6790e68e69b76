"""torchrun worker: the multi-GPU push exchange, bit-exact per rank against the oracle.

    torchrun --nproc-per-node N tests/mgpu_worker.py [config] [projector]

Every rank plans the whole step on its GPU, pushes its loader rows into the
encoder ranks' receive windows over NVLink, runs the stand-in encoder, and
pushes the returned rows into their LLM ranks' packed buffers.  Each rank then
checks its own receive windows and LLM buffer against the fake-world oracle
(which every rank can compute: all inputs are seeded).
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import dataplane as odp  # noqa: E402
from oracle import cphybrid as ocph  # noqa: E402
from oracle import lssp as olssp  # noqa: E402
from oracle import planner as oplan  # noqa: E402
from oracle import workload as owork  # noqa: E402
from paper_2605_08962_b200 import configs, planner  # noqa: E402
from paper_2605_08962_b200.dataplane import MuxPath  # noqa: E402


def payload(rows, width, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randn(max(rows, 1), width, generator=g).to(torch.bfloat16)


def run_overlapped(path, name, cfg, world, rank, dev, gbs, dp, sp, d_in, d_llm, proj=None):
    """MuxPath.run_pipeline with overlap_dispatch: step k+1's dispatch under step
    k's return, 4 chained steps; each step's receive windows (captured in the
    encoder slot) and LLM buffer checked bit-exactly — or, with proj = (Ws, bs,
    d_enc), the projected rows against an fp32 reference (the bench's default
    multi-GPU path: pair GEMM, fused signal, overlapped dispatch).  Returns failures."""
    descs = owork.descs_from_config(configs.DATASETS, cfg["datasets"])
    carry, seen, steps, oracle = None, {}, [], []
    for step in range(4):
        _, rest, drawn, chunks = owork.generate(descs, cfg["phases"], False, step, cfg["seed"],
                                                gbs, dp, 1, configs.CAPACITY,
                                                carry if cfg["carry"] else None)
        for s in drawn:
            seen[s[0]] = s[1]
        t = oplan.step_table(list(carry or []) if cfg["carry"] else [], drawn, chunks, seen)
        carry = rest
        o = oplan.plan_step(t, configs.CAPACITY, gbs, dp, sp, world, 1, path.method)
        arenas = [[payload(int(o["arena_rows"][r, g]), d_in[g], 7000 + 100 * step + 10 * r + g)
                   for g in range(2)] for r in range(world)]
        table = planner.StepTable(t["lens"].astype(np.int32), t["mods"].astype(np.int32),
                                  t["ids"], t["carry_seq"].astype(np.int32),
                                  t["n_carry_seqs"], np.asarray(t["chunk_off"], np.int32))
        steps.append((planner.DeviceTable(table, dev), [a.to(dev) for a in arenas[rank]]))
        oracle.append((t, o, arenas))
    recv_got, llm_got = [], []

    def encoder(k, p, s):
        o = oracle[k][1]
        recv_got.append([path.recv_view(g, int(o["recv_rows"][rank, g])).clone()
                         for g in range(2)])
        path.encode_standin(p, steps[k][0], s)

    def after(k, p, s):
        path.check_wait()
        llm_got.append(path.llm_view(int(oracle[k][1]["llm_rows"][rank])).clone())

    path.zero_llm()
    torch.cuda.synchronize()
    dist.barrier()
    path.run_pipeline(steps, encoder=encoder, after_step=after)
    path.finish()
    torch.cuda.synchronize()
    fails = 0
    for k, (t, o, arenas) in enumerate(oracle):
        ar = [[a.view(torch.int16).numpy().view(np.uint16) for a in arenas[r]]
              for r in range(world)]
        recv, _, llm = odp.run_world(o, t, world, ar, d_in, (d_llm, d_llm), d_llm)
        for g in range(2):
            got = recv_got[k][g].cpu().view(torch.int16).numpy().view(np.uint16)
            if not np.array_equal(got, recv[rank][g]):
                print(f"rank {rank} overlapped step {k}: recv group {g} differs", flush=True)
                fails += 1
        # LLM buffers alternate between steps and are not cleared: compare the rows
        # this step writes (text rows are not part of the return)
        mask = np.zeros(int(o["llm_rows"][rank]), bool)
        for (i, src, dst_rank, dst_row, rows) in o["pieces"]:
            if dst_rank == rank:
                mask[dst_row:dst_row + rows] = True
        if proj is not None:
            Ws, bs, d_enc = proj
            ref = torch.zeros(len(mask), d_llm, device=dev)
            for (i, src, dst_rank, dst_row, rows) in o["pieces"]:
                if dst_rank != rank:
                    continue
                g = int(o["group"][i])
                x = torch.from_numpy(odp.standin(int(t["ids"][i]), int(t["lens"][i]), d_enc[g])
                                     .view(np.int16)).view(torch.bfloat16).to(dev)[:rows]
                ref[dst_row:dst_row + rows] = x.float() @ Ws[g].to(dev).float().t() + \
                    bs[g].to(dev).float()
            m = torch.from_numpy(mask).to(dev)
            err = (llm_got[k].float()[m] - ref[m]).abs()
            if not bool((err <= 2.0 ** -7 * ref[m].abs() + 1e-3).all()):
                print(f"rank {rank} overlapped step {k}: projected rows differ", flush=True)
                fails += 1
        else:
            got = llm_got[k].cpu().view(torch.int16).numpy().view(np.uint16)
            if not np.array_equal(got[mask], llm[rank][mask]):
                print(f"rank {rank} overlapped step {k}: llm rows differ", flush=True)
                fails += 1
        if rank == 0:
            print(f"overlapped step {k}: {int(o['recv_rows'].sum())} modality tokens ok="
                  f"{fails == 0}", flush=True)
    return fails


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    narrow = "narrow" in sys.argv
    proj = "proj" in sys.argv
    lssp = "lssp" in sys.argv  # LSSP eta split: long samples sharded over encoder groups
    cp = "cp" in sys.argv  # CpHybrid LLM placement instead of Ulysses shards
    overlap = "overlap" in sys.argv  # run_pipeline with the overlapped dispatch
    meta = "meta" in sys.argv  # step table from the decentralized metadata all-gather
    rg = 2 if "rg2" in sys.argv else 0  # reorder groups of two ranks
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = configs.CONFIGS[name]
    sp = cfg["sp"] if world % cfg["sp"] == 0 and world >= cfg["sp"] else 1
    dp = world // sp
    gbs = cfg["gbs_per_replica"] * dp
    full = "full" in sys.argv  # the bench's real widths (d_enc 1280, d_llm 4096)
    d_in = (20, 8) if narrow else configs.D_IN
    d_llm = 64 if narrow else (configs.D_LLM if full else 512)
    descs = owork.descs_from_config(configs.DATASETS, cfg["datasets"])
    carry, seen = None, {}
    d_enc = tuple(configs.D_ENC) if full else (256, 256)
    if proj and sp != 1:
        sp, dp = 1, world
        gbs = cfg["gbs_per_replica"] * dp
    path = MuxPath(capacity=configs.CAPACITY, gbs=gbs, dp=dp, sp=sp, world=world, rank=rank,
                   d_in=d_in, d_enc=d_enc, d_llm=d_llm, device=dev, group=dist.group.WORLD,
                   projector=proj,
                   projector_return="staged" if "staged" in sys.argv else "fused",
                   lssp_eta=2048 if lssp else None, lssp_sp=world if lssp else 1,
                   reshard="cp_hybrid" if cp else "ulysses", cp_threshold=2048 if cp else 0,
                   overlap_dispatch=overlap, reorder_group=rg)
    if proj:
        gw = torch.Generator().manual_seed(9)
        Ws = [(torch.randn(d_llm, d_enc[g], generator=gw) / d_enc[g] ** 0.5).to(torch.bfloat16)
              for g in range(2)]
        bs = [torch.randn(d_llm, generator=gw).to(torch.bfloat16) for g in range(2)]
        for g in range(2):
            path.set_projector(g, Ws[g].to(dev), bs[g].to(dev))
    if overlap:
        path.method = "lpt_local"
        fails = run_overlapped(path, name, cfg, world, rank, dev, gbs, dp, sp, d_in, d_llm,
                               (Ws, bs, d_enc) if proj else None)
        t = torch.tensor([fails], device=dev)
        dist.all_reduce(t)
        dist.destroy_process_group()
        sys.exit(1 if int(t.item()) else 0)
    fails = 0
    for step in range(3):
        _, rest, drawn, chunks = owork.generate(descs, cfg["phases"], False, step, cfg["seed"],
                                                gbs, dp, 1, configs.CAPACITY,
                                                carry if cfg["carry"] else None)
        for s in drawn:
            seen[s[0]] = s[1]
        t = oplan.step_table(list(carry or []) if cfg["carry"] else [], drawn, chunks, seen)
        carry = rest
        for method in (("lpt_local",) if proj else ("lpt", "kk", "lpt_local")):
            path.method = method
            o = oplan.plan_step(t, configs.CAPACITY, gbs, dp, sp, world, 1, method,
                                reorder_group=rg)
            if cp:
                o = ocph.place(o, t, gbs, dp, sp, configs.CAPACITY, 2048)
            lay = None
            if lssp:  # group of all ranks on even steps, pairs on odd steps
                path.lssp_sp = world if step % 2 == 0 else 2
                lay = olssp.layout(o, t["lens"], world, path.lssp_eta, path.lssp_sp)
            arenas = [[payload(int(o["arena_rows"][r, g]), d_in[g], 1000 * step + 10 * r + g)
                       for g in range(2)] for r in range(world)]
            table = planner.StepTable(t["lens"].astype(np.int32), t["mods"].astype(np.int32),
                                      t["ids"], t["carry_seq"].astype(np.int32),
                                      t["n_carry_seqs"], np.asarray(t["chunk_off"], np.int32))
            if meta:  # decentralized loaders: this rank's share + the metadata all-gather
                dtab = planner.gather_table(table.shard(rank, world), dev, dist.group.WORLD)
                assert np.array_equal(dtab.blob.cpu().numpy()[:table.blob().size], table.blob())
                table = dtab.table
            else:
                dtab = planner.DeviceTable(table, dev)
            plan = path.plan(dtab)
            plan.check(table)
            path.zero_llm()
            torch.cuda.synchronize()
            dist.barrier()
            path.dispatch(plan, [a.to(dev) for a in arenas[rank]])
            path.encode_standin(plan, dtab)
            path.return_scatter(plan)
            path.finish()
            torch.cuda.synchronize()
            path.check_wait()
            ar = [[a.view(torch.int16).numpy().view(np.uint16) for a in arenas[r]]
                  for r in range(world)]
            if proj:  # projected rows vs a torch fp32 reference (tolerance, test_gpu_proj.py)
                n = int(o["llm_rows"][rank])
                got = path.llm_view(n).float()
                ref = torch.zeros(n, d_llm, device=dev)
                mask = torch.zeros(n, dtype=torch.bool, device=dev)
                for (i, src, dst_rank, dst_row, rows) in o["pieces"]:
                    if dst_rank != rank:
                        continue
                    g = int(o["group"][i])
                    x = torch.from_numpy(odp.standin(int(t["ids"][i]), int(t["lens"][i]), d_enc[g])
                                         .view(np.int16)).view(torch.bfloat16).to(dev)
                    ref[dst_row:dst_row + rows] = x.float() @ Ws[g].to(dev).float().t() + \
                        bs[g].to(dev).float()
                    mask[dst_row:dst_row + rows] = True
                err = (got - ref).abs()
                ok = bool((err <= 2.0 ** -7 * ref.abs() + 1e-3).all()) and \
                    bool((got[~mask] == 0).all())
                if not ok:
                    print(f"rank {rank} step {step}: projected rows differ", flush=True)
                    fails += 1
                dist.barrier()
                continue
            if lay is None:
                recv, _, llm = odp.run_world(o, t, world, ar, d_in, (d_llm, d_llm), d_llm)
                rows_of = o["recv_rows"]
            else:
                recv, _, llm = olssp.run_world(o, lay, t, world, ar, d_in, (d_llm, d_llm), d_llm)
                rows_of = lay["recv_rows"]
            for g in range(2):
                n = int(rows_of[rank, g])
                got = path.recv_view(g, n).cpu().view(torch.int16).numpy().view(np.uint16)
                if not np.array_equal(got, recv[rank][g]):
                    print(f"rank {rank} step {step} {method}: recv group {g} differs", flush=True)
                    fails += 1
            n = int(o["llm_rows"][rank])
            got = path.llm_view(n).cpu().view(torch.int16).numpy().view(np.uint16)
            if not np.array_equal(got, llm[rank]):
                print(f"rank {rank} step {step} {method}: llm buffer differs", flush=True)
                fails += 1
            # gradient return: every rank's dY rows back to the encoder ranks
            dys = [payload(max(int(o["llm_rows"][r]), 1), d_llm, 5000 + 10 * step + r)
                   for r in range(world)]
            dist.barrier()
            path.grad_return(plan, dys[rank].to(dev))
            torch.cuda.synchronize()
            path.check_wait()
            dyh = [d.view(torch.int16).numpy().view(np.uint16) for d in dys]
            want = odp.run_grad(o, world, dyh, d_llm) if lay is None else \
                olssp.run_grad(lay, world, dyh, d_llm)
            for g in range(2):
                r_ = int(rows_of[rank, g])
                got = path.grad_view(g, r_).cpu().view(torch.int16).numpy().view(np.uint16)
                if not np.array_equal(got, want[rank][g]):
                    print(f"rank {rank} step {step} {method}: gradient group {g} differs",
                          flush=True)
                    fails += 1
            moved = int(o["recv_rows"].sum())
            if rank == 0:
                print(f"step {step} {method}: {moved} modality tokens over {world} ranks ok="
                      f"{fails == 0}", flush=True)
            dist.barrier()
    t = torch.tensor([fails], device=dev)
    dist.all_reduce(t)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
