"""Device planner latency per step table size: cfg5 tables at world 1..8 (one GPU,
every rank's plan is the same computation), CUDA events, median of 20."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_08962_b200 import configs, planner  # noqa: E402

for name in ("cfg2", "cfg5", "target1"):
    for world in (1, 2, 4, 8):
        cfg, dp, sp, gbs = bench.workload(name, world)
        tabs = bench.generate_steps(name, world, 3)
        ts = []
        for t in tabs:
            d = planner.DeviceTable(t, "cuda")
            c = planner.make_cfg(t, configs.CAPACITY, gbs, dp, sp, world, 1, "lpt_local", False,
                                 0, row_bytes_in=(1176, 1024), row_bytes_ret=(8192, 8192))
            p = planner.plan_step(d, c)
            p.check(t)
            for _ in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                planner.plan_step(d, c, p)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
        print(f"{name} world {world}: S {tabs[0].S}-{tabs[-1].S}, plan {np.median(ts):.1f} us "
              f"(min {min(ts):.1f})", flush=True)
