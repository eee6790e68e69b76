"""Mixed local + NVLink exchange, the shape of cfg5's return at N GPUs:

  torchrun --nproc-per-node N scripts/nvlink_probe3.py [local_MiB] [remote_MiB_per_peer]

One launch of mux_copy_ranges (SM stores, 32 KiB chunks dealt round-robin over the
ranges) for: A local copy only, B pushes to every peer only, C both in one launch,
D both as two concurrent launches on two streams.  Max-over-ranks CUDA-event ms."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08962_b200 import _lib  # noqa: E402
from paper_2605_08962_b200.dataplane import _Window  # noqa: E402


def main():
    lm = int(sys.argv[1]) if len(sys.argv) > 1 else 170
    rm = int(sys.argv[2]) if len(sys.argv) > 2 else 14
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    nl, nr = lm << 20, rm << 20
    src = torch.empty(nl + world * nr, dtype=torch.uint8, device=dev).fill_(rank)
    dstl = torch.empty(nl, dtype=torch.uint8, device=dev)
    win = _Window(world * nr, dev, dist.group.WORLD, world)
    L = _lib.lib()
    s1 = torch.cuda.current_stream()
    s2 = torch.cuda.Stream(dev)

    def ranges(pairs):
        t = [torch.tensor([p[i] for p in pairs], dtype=torch.int64, device=dev) for i in range(3)]
        return t + [max(p[2] for p in pairs), len(pairs)]

    loc = [(dstl.data_ptr(), src.data_ptr(), nl)]
    rem = [(win.ptrs[r] + rank * nr, src.data_ptr() + nl + r * nr, nr)
           for r in range(world) if r != rank]
    A, B, Cm = ranges(loc), ranges(rem), ranges(rem + loc)

    def go(rg, stream, grid=0, mode=0):
        d, sr, b, mx, n = rg
        if n == 0 or mx == 0:
            return
        _lib.check(L.mux_copy_ranges(n, d.data_ptr(), sr.data_ptr(), b.data_ptr(), mx, grid,
                                     mode, stream.cuda_stream))

    def fork(remote_fn, local_grid=888):
        ev = torch.cuda.Event()
        ev.record(s1)
        s2.wait_event(ev)
        remote_fn()
        go(A, s1, local_grid)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s1.wait_event(ev2)

    def both():
        fork(lambda: go(B, s2, 296))

    def both_tma(grid):
        return lambda: fork(lambda: go(B, s2, grid, 1))

    def both_ce():
        def ce():
            for (d, sr, n) in rem:
                if n:
                    _lib.check(L.mux_memcpy_async(d, sr, n, s2.cuda_stream))
        fork(ce, 1184)

    out = {"world": world, "local_mib": lm, "remote_mib_per_peer": rm}
    for nm, fn in (("A_local", lambda: go(A, s1)), ("B_remote", lambda: go(B, s1)),
                   ("B_remote_tma", lambda: go(B, s1, 296, 1)),
                   ("C_mixed_one_launch", lambda: go(Cm, s1)), ("D_two_streams", both),
                   ("E_remote_tma148_local_sm", both_tma(148)),
                   ("E_remote_tma296_local_sm", both_tma(296)),
                   ("F_remote_copy_engine_local_sm", both_ce)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1)
        for _ in range(10):
            fn()
        b.record(s1)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 10], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[nm + "_ms"] = round(float(t.item()), 4)
        dist.barrier()
    out["remote_gbs_in_B"] = round((world - 1) * nr / out["B_remote_ms"] / 1e6, 1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    win.handle.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
