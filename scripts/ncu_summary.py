"""Summarise an ncu report (--set full or the launch list) into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_prof.md
    python scripts/ncu_summary.py gpurun_out/launches.csv profiles/r01_launches.md
"""

import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: {path}", ""]
    for d in data:
        name = d[hdr.index("Kernel Name")][:90]
        lines.append(f"## {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"- {k}: {d[i]} {units[i]}")
        lines.append("")
    return "\n".join(lines)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = {}
    lines = [f"# launch list (gpu__time_duration.sum, --clock-control none): {path}", "",
             "| # | kernel | duration |", "|---|---|---|"]
    for n, r in enumerate(data):
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(r[ui], 1.0)
        tot[name] = tot.get(name, 0.0) + v * scale
        lines.append(f"| {n} | {name} | {r[vi]} {r[ui]} |")
    s = sum(tot.values())
    lines += ["", "| kernel | total us | share |", "|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda t: -t[1]):
        lines.append(f"| {k} | {v:.1f} | {v / s:.1%} |")
    return "\n".join(lines)


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    text = rep(src) if src.endswith(".ncu-rep") else launches(src)
    open(dst, "w").write(text + "\n")
    print(text[:3000])
