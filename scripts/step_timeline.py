"""Per-kernel CUDA-event timeline of the data path on every rank (no profiler).

    torchrun --nproc-per-node N scripts/step_timeline.py [config] [steps]

Each step is issued eagerly with an event between every launch, so each
interval is one kernel (or one flag wait).  Prints, per rank, the mean
microseconds per interval over the steps.
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08962_b200 import _lib, configs  # noqa: E402
from paper_2605_08962_b200.dataplane import N_GROUPS, MuxPath  # noqa: E402
from paper_2605_08962_b200.planner import DeviceTable, _stream_ptr  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
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
    tables = bench.generate_steps(name, world, 4)
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
        pl = path.plan(d)
        path.encode_standin(pl, d)  # realistic encoder rows (GEMM power is data-dependent)
        info = pl.host()
        arenas.append([torch.randn(max(int(info["arena_rows"][rank, g]), 1), configs.D_IN[g],
                                   device=dev).to(torch.bfloat16) for g in range(2)])
    L = _lib.lib()
    st = torch.cuda.current_stream()
    s = _stream_ptr(st)
    names = []
    acc = []

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    for k in range(steps + 3):
        i = k % len(dtabs)
        marks = [("start", ev())]
        p = path.plan(dtabs[i], st)
        marks.append(("plan", ev()))
        tbl = path._arena_table(arenas[i])
        if world == 1:
            L.mux_segcopy(C.byref(p.cfg), p.ptr, 0, tbl.data_ptr(), path.recv_dst.data_ptr(), 0,
                          path.sync.data_ptr(), s)
            marks.append(("dispatch copy", ev()))
        else:
            L.mux_segcopy_signal(C.byref(p.cfg), p.ptr, 0, tbl.data_ptr(),
                                 path.recv_dst.data_ptr(), 0, path.flag_ptrs.data_ptr(),
                                 path.sync.data_ptr(), path.epoch_ctr.data_ptr(), s)
            marks.append(("dispatch copy", ev()))
            L.mux_wait(world, path.flags.tensor.data_ptr(), path.epoch_ctr.data_ptr(), 20000,
                       path.wait_err.data_ptr(), s)
            marks.append(("dispatch wait", ev()))
        if not proj:
            if world == 1:
                L.mux_segcopy(C.byref(p.cfg), p.ptr, 1, path.enc_src.data_ptr(),
                              path.llm_dst[0].data_ptr(), 0, path.sync[2:].data_ptr(), s)
                marks.append(("return copy", ev()))
            else:
                dst = path.llm_dst[0]
                if os.environ.get("MUX_TIMELINE_LOCAL"):  # experiment: every row stays local
                    dst = torch.full_like(dst, int(path.llm_bufs[0].ptrs[rank]))
                if os.environ.get("MUX_TIMELINE_PLAIN"):  # experiment: local, non-VMM buffer
                    if not hasattr(path, "_plain"):
                        path._plain = torch.empty_like(path.llm_bufs[0].tensor)
                    dst = torch.full_like(dst, int(path._plain.data_ptr()))
                if os.environ.get("MUX_TIMELINE_RING"):  # experiment: every row to rank+1
                    dst = torch.full_like(dst, int(path.llm_bufs[0].ptrs[(rank + 1) % world]))
                L.mux_segcopy_signal(C.byref(p.cfg), p.ptr, 1, path.enc_src.data_ptr(),
                                     dst.data_ptr(), 0, path.flag_ptrs.data_ptr(),
                                     path.sync[2:].data_ptr(), path.epoch_ctr.data_ptr(), s)
                marks.append(("return copy", ev()))
                L.mux_wait(world, path.flags.tensor.data_ptr(), path.epoch_ctr.data_ptr(), 20000,
                           path.wait_err.data_ptr(), s)
                marks.append(("return wait", ev()))
        elif world == 1 or path.ret_mode == _lib.RET_FINAL:
            path._row_map(p, path.row_dst, st)
            if os.environ.get("MUX_TIMELINE_LOCAL"):  # experiment: every store local
                path.row_dst.bitwise_and_((1 << 40) - 1).bitwise_or_(rank << 40)
            marks.append(("row map", ev()))
            hdr = p.ptr + p.layout.header
            groups = (_lib.ProjGroup * N_GROUPS)()
            for g in range(N_GROUPS):
                groups[g] = _lib.ProjGroup(path.enc_out[g].data_ptr(), path.weight[g].data_ptr(),
                                           0, path.max_rows, hdr + 8 * (_lib.H_RECV_ROWS0 + g),
                                           path.d_enc[g], 0,
                                           path.row_dst.data_ptr() + 8 * g * path.max_rows)
            L.mux_proj_scatter_grouped(groups, N_GROUPS, path.d_llm, path.llm_dst[0].data_ptr(),
                                       int(os.environ.get("MUX_GEMM_CTAS", "0")), s)
            marks.append(("projector GEMM", ev()))
            if world > 1:
                L.mux_signal(rank, world, path.flag_ptrs.data_ptr(), path.epoch_ctr.data_ptr(), s)
                marks.append(("signal", ev()))
                L.mux_wait(world, path.flags.tensor.data_ptr(), path.epoch_ctr.data_ptr(), 20000,
                           path.wait_err.data_ptr(), s)
                marks.append(("return wait", ev()))
            p.row_map = None
        else:
            L.mux_segcopy_signal(C.byref(p.cfg), p.ptr, 1, path.enc_src.data_ptr(),
                                 path.stage_dst[0].data_ptr(), 0, path.flag_ptrs.data_ptr(),
                                 path.sync[2:].data_ptr(), path.epoch_ctr.data_ptr(), s)
            marks.append(("return copy (d_enc rows)", ev()))
            L.mux_wait(world, path.flags.tensor.data_ptr(), path.epoch_ctr.data_ptr(), 20000,
                       path.wait_err.data_ptr(), s)
            marks.append(("return wait", ev()))
            hdr = p.ptr + p.layout.header
            for g in range(N_GROUPS):
                L.mux_stage_rows(C.byref(p.cfg), p.ptr, p.lens_ptr, g, path.row_dst.data_ptr(),
                                 path.max_llm_rows, s)
                marks.append((f"stage_rows g{g}", ev()))
                L.mux_proj_scatter_dev(path.stage[0][g].tensor.data_ptr(),
                                       path.weight[g].data_ptr(), 0, path.max_llm_rows,
                                       hdr + 8 * (_lib.H_STAGE_ROWS0 + g), path.d_enc[g],
                                       path.d_llm, path.row_dst.data_ptr(),
                                       path.llm_dst[0].data_ptr(), 0, s)
                marks.append((f"GEMM g{g}", ev()))
        torch.cuda.synchronize()
        if k >= 3:
            names = [m[0] for m in marks[1:]]
            acc.append([a[1].elapsed_time(b[1]) * 1e3 for a, b in zip(marks, marks[1:])])
    mean = np.mean(np.array(acc), axis=0).tolist()
    rows = [[int(x) for x in path.plan(d).host()["recv_rows"][rank]] for d in dtabs]
    out = {"rank": rank, "world": world, "config": name,
           "us": {n: round(v, 1) for n, v in zip(names, mean)}, "recv_rows": rows}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
