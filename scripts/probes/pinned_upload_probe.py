"""Per-buffer H2D copy-engine time for the e2e loader's pinned arenas: eight
pinned host buffers made the way bench.py's e2e makes them (device tensor ->
.cpu() -> .pin_memory()), uploaded to one device slot in order, twice, with
CUDA events around every copy.  Separates a slow first DMA from one buffer
(host-memory / IOMMU effect) from anything in the pipeline around it."""

import json

import torch

SIZES_MB = [61.7, 58.4, 46.7, 39.1, 51.4, 43.4, 52.4, 51.9]  # cfg2's eight distinct steps


def main():
    dev = torch.device("cuda", 0)
    host = []
    for mb in SIZES_MB:
        n = int(mb * 1e6) // 2
        host.append(torch.randn(n, device=dev).to(torch.bfloat16).cpu().pin_memory())
    slot = torch.empty(max(h.numel() for h in host), dtype=torch.bfloat16, device=dev)
    up = torch.cuda.Stream(dev)
    out = {}
    for rnd, order in (("warm", [0, 1, 2]), ("first", list(range(8))),
                       ("second", list(range(8))), ("third", list(range(8)))):
        evs = []
        for i in order:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(up):
                a.record(up)
                slot[: host[i].numel()].copy_(host[i], non_blocking=True)
                b.record(up)
            evs.append((i, a, b))
        torch.cuda.synchronize()
        out[rnd] = {i: round(host[i].numel() * 2 / a.elapsed_time(b) / 1e6, 1) for i, a, b in evs}
    print(json.dumps({"h2d_gbs_per_buffer": out}))


if __name__ == "__main__":
    main()
