"""Copy-engine A/B over NVLink (one process per GPU):

  torchrun --nproc-per-node N scripts/nvlink_probe2.py [MiB]

Every rank pushes MiB in one launch of mux_copy_ranges: ring (all to the next
rank) or all-to-all (MiB split evenly over the other ranks, all written at
once), with SM stores (mode 0, the segment-copy engine) or TMA bulk copies
(mode 1); the copy engine (cudaMemcpyAsync) ring; and a local HBM copy by
each mode.  Max-over-ranks CUDA-event time; one JSON line from rank 0."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08962_b200 import _lib  # noqa: E402
from paper_2605_08962_b200.dataplane import _Window  # noqa: E402


def timed(fn, dev, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) / 1e3


def main():
    mib = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    n = mib << 20
    out = {"world": world, "bytes_per_rank": n}
    x = torch.empty(n, dtype=torch.uint8, device=dev).fill_(rank)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
    win = _Window(n, dev, dist.group.WORLD, world)
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream

    def ranges(pairs):
        d = torch.tensor([p[0] for p in pairs], dtype=torch.int64, device=dev)
        sr = torch.tensor([p[1] for p in pairs], dtype=torch.int64, device=dev)
        b = torch.tensor([p[2] for p in pairs], dtype=torch.int64, device=dev)
        return d, sr, b, max(p[2] for p in pairs), len(pairs)

    share = (n // max(world - 1, 1)) & ~4095
    pats = {"ring": ranges([(win.ptrs[(rank + 1) % world], x.data_ptr(), n)]),
            "alltoall": ranges([(win.ptrs[r] + rank * share % max(n - share, 1),
                                 x.data_ptr() + (r if r < rank else r - 1) * share, share)
                                for r in range(world) if r != rank]),
            "local": ranges([(y.data_ptr(), x.data_ptr(), n)])}
    for nm, (d, sr, b, mx, cnt) in pats.items():
        moved = n if nm != "alltoall" else share * cnt
        for mode, grids in ((0, (0,)), (1, (148, 296, 592))):
            for g in grids:
                t = timed(lambda: _lib.check(L.mux_copy_ranges(cnt, d.data_ptr(), sr.data_ptr(),
                                                               b.data_ptr(), mx, g, mode, s)),
                          dev)
                gbs = moved / t / 1e9 * (2 if nm == "local" else 1)
                out[f"{nm}_{'sm' if mode == 0 else 'tma'}{'' if not g else '_g' + str(g)}_gbs"] = \
                    round(gbs, 1)
    t = timed(lambda: _lib.check(L.mux_memcpy_async(win.ptrs[(rank + 1) % world], x.data_ptr(),
                                                    n, s)), dev)
    out["ring_copy_engine_gbs"] = round(n / t / 1e9, 1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    win.handle.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
