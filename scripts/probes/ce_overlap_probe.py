"""Does a copy-engine NVLink push overlap an SM-driven local copy better than
SM pushes do?  (cfg5's exchange: each rank copies ~156-185 MB locally and pushes
~13-67 MB to peers in the same kernel, and takes about the SUM of the two
alone.)  Under torchrun, every rank, max over ranks of CUDA-event time:
  local     SM copy of L bytes inside HBM (mux_copy_bytes)
  sm_push   SM push of R bytes to rank+1 (mux_copy_bytes to the peer window)
  ce_push   copy-engine push of R bytes to rank+1 (cudaMemcpyAsync)
  local+sm  both SM copies concurrently (two streams)
  local+ce  SM local copy and copy-engine push concurrently (two streams)
  tma_push, local+tma[G]   the push by TMA bulk copies (mux_copy_ranges mode 1)
  sm+ce_push, ce+ce_push   two R-byte pushes to the peer at once (aggregate link rate)

  torchrun --nproc-per-node 2 scripts/probes/ce_overlap_probe.py
"""

import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2605_08962_b200 import _lib  # noqa: E402
from paper_2605_08962_b200.dataplane import _Window  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()
    LB, RB = 160 << 20, 48 << 20
    win = _Window(2 * RB, dev, dist.group.WORLD, world)
    src_l = torch.empty(LB, dtype=torch.uint8, device=dev).fill_(1)
    dst_l = torch.empty(LB, dtype=torch.uint8, device=dev)
    src_r = torch.empty(RB, dtype=torch.uint8, device=dev).fill_(2)
    peer = win.ptrs[(rank + 1) % world]
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def local(s):
        _lib.check(L.mux_copy_bytes(dst_l.data_ptr(), src_l.data_ptr(), LB, 0, s.cuda_stream))

    def sm_push(s, grid=0):
        _lib.check(L.mux_copy_bytes(C.c_void_p(peer), src_r.data_ptr(), RB, grid, s.cuda_stream))

    rng = [torch.tensor([v], dtype=torch.int64, device=dev)
           for v in (peer, src_r.data_ptr(), RB)]

    def tma_push(s, grid=0):
        _lib.check(L.mux_copy_ranges(1, rng[0].data_ptr(), rng[1].data_ptr(), rng[2].data_ptr(),
                                     RB, grid, 1, s.cuda_stream))

    def ce_push(s, off=0):
        _lib.check(L.mux_memcpy_async(C.c_void_p(peer + off), src_r.data_ptr(), RB,
                                      s.cuda_stream))

    cases = {
        "local": lambda: local(s1),
        "sm_push": lambda: sm_push(s1),
        "ce_push": lambda: ce_push(s1),
        "local+sm": lambda: (local(s1), sm_push(s2)),
        "local+sm148": lambda: (local(s1), sm_push(s2, 148)),
        "local+ce": lambda: (local(s1), ce_push(s2)),
        "sm+ce_push": lambda: (sm_push(s1), ce_push(s2, RB)),  # 2 x RB to the peer
        "ce+ce_push": lambda: (ce_push(s1), ce_push(s2, RB)),
        "tma_push": lambda: tma_push(s1),
        "local+tma": lambda: (local(s1), tma_push(s2)),
        "local+tma148": lambda: (local(s1), tma_push(s2, 148)),
        "local+tma32": lambda: (local(s1), tma_push(s2, 32)),
        "local+sm32": lambda: (local(s1), sm_push(s2, 32)),
    }
    out = {"local_bytes": LB, "remote_bytes": RB}
    main_s = torch.cuda.current_stream()
    for name, fn in cases.items():
        best = None
        for rep in range(4):
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            s1.wait_event(a)
            s2.wait_event(a)
            fn()
            e1, e2 = torch.cuda.Event(), torch.cuda.Event()
            e1.record(s1)
            e2.record(s2)
            main_s.wait_event(e1)
            main_s.wait_event(e2)
            b.record(main_s)
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rep:
                best = float(t.item()) if best is None else min(best, float(t.item()))
        out[name + "_ms"] = round(best, 4)
    if rank == 0:
        print(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
