"""NVLink denominators on this box, one process per GPU:

  torchrun --nproc-per-node N scripts/nvlink_probe.py [MiB]

1. NCCL all_to_all_single, uniform, MiB per rank: algorithm and bus bandwidth;
2. our copy kernel pushing MiB into the next rank's symmetric window (all ranks at
   once, ring pattern), and the same bytes split evenly over all peers;
3. cudaMemcpyAsync (copy engine) to the next rank's window, for comparison.
Prints one JSON line from rank 0; every number is max-over-ranks device time.
"""
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
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    y = torch.empty(n, dtype=torch.uint8, device=dev)
    t = timed(lambda: dist.all_to_all_single(y, x), dev)
    out["nccl_alltoall_algbw_gbs"] = n / t / 1e9
    out["nccl_alltoall_busbw_gbs"] = n * (world - 1) / world / t / 1e9
    win = _Window(n, dev, dist.group.WORLD, world)
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    peer = win.ptrs[(rank + 1) % world]
    t = timed(lambda: _lib.check(L.mux_copy_bytes(peer, x.data_ptr(), n, 0, s)), dev)
    out["kernel_push_ring_gbs"] = n / t / 1e9
    share = (n // world) & ~255

    def spread():
        for r in range(world):
            if r != rank:
                _lib.check(L.mux_copy_bytes(win.ptrs[r] + rank * share, x.data_ptr() + r * share,
                                            share, 0, s))
    t = timed(spread, dev)
    out["kernel_push_alltoall_gbs"] = share * (world - 1) / t / 1e9
    t = timed(lambda: _lib.check(L.mux_memcpy_async(peer, x.data_ptr(), n, s)), dev)
    out["copy_engine_push_ring_gbs"] = n / t / 1e9
    t = timed(lambda: _lib.check(L.mux_copy_bytes(y.data_ptr(), x.data_ptr(), n, 0, s)), dev)
    out["kernel_local_copy_gbs"] = 2 * n / t / 1e9
    if rank == 0:
        print(json.dumps(out), flush=True)
    win.handle.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
