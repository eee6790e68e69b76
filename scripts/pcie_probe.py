"""Host<->device bandwidth probe: copy engine (cudaMemcpyAsync, 1 or 2 streams)
against SM-driven reads of pinned host memory (mux_copy_bytes over UVA).
Decides whether the loader upload can be fused into the pack kernel."""

import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2605_08962_b200 import _lib  # noqa: E402


def timed(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


def main():
    L = _lib.lib()
    n = 64 << 20
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    host.random_(0, 255)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    s2 = torch.cuda.Stream()
    out = {}
    out["ce_h2d_1stream"] = n / timed(lambda: dev.copy_(host, non_blocking=True)) / 1e9

    def two():
        h = n // 2
        ev = torch.cuda.Event()
        ev.record(st)
        s2.wait_event(ev)
        dev[:h].copy_(host[:h], non_blocking=True)
        with torch.cuda.stream(s2):
            dev[h:].copy_(host[h:], non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        st.wait_event(ev2)
    out["ce_h2d_2streams"] = n / timed(two) / 1e9
    out["ce_d2h_1stream"] = n / timed(lambda: host.copy_(dev, non_blocking=True)) / 1e9
    for grid in (148, 296, 592, 1184, 2368):
        def k():
            _lib.check(L.mux_copy_bytes(dev.data_ptr(), host.data_ptr(), n, grid,
                                        st.cuda_stream), "copy")
        out[f"sm_h2d_grid{grid}"] = n / timed(k) / 1e9
    assert torch.equal(dev.cpu(), host)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
