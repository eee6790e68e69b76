"""Phase timing of the device planner from its globaltimer stamps (header 16..26)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_08962_b200 import configs  # noqa: E402
from paper_2605_08962_b200.dataplane import MuxPath  # noqa: E402
from paper_2605_08962_b200.planner import DeviceTable  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "target1"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg, dp, sp, gbs = bench.workload(name, world)
tables = bench.generate_steps(name, world, 4)
path = MuxPath(capacity=configs.CAPACITY, gbs=gbs, dp=dp, sp=sp, world=world, rank=0,
               d_in=configs.D_IN, d_llm=configs.D_LLM, max_rows=gbs * configs.CAPACITY)
names = ["ffd(start->fin start)", "A-B", "C", "D", "E", "F", "G (assign)", "H", "H2+I (segments)"]
acc = []
for rep in range(20):
    for t in tables:
        dt = DeviceTable(t, "cuda")
        p = path.plan(dt)
        torch.cuda.synchronize()
        h = p.header()
        ts = [h[20 + x - 16] for x in (16, 17, 18, 19, 20, 21, 22, 23, 24, 25)]
        acc.append(np.diff(np.array(ts, dtype=np.float64)) / 1e3)
a = np.array(acc[8:])
print(f"{name} world={world}: S={[t.S for t in tables]}")
for nm, v in zip(names, a.mean(0)):
    print(f"  {nm:24s} {v:8.2f} us")
print(f"  total (ffd start -> end) {a.sum(1).mean():8.2f} us")
