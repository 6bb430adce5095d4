"""Summarise ncu captures for profiles/: the launch list (gpu__time_duration per kernel, --clock-control none) and
the key counters of each `ncu --set full` capture (DRAM bytes, PCIe bytes, sysmem sectors, duration, occupancy).

  python tools/ncu_summary.py OUT.md --launches gpurun_out/launches.csv --full gpurun_out/prof_staged.ncu-rep ...
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__bytes.sum.per_second", "dram B/s"),
    ("pcie__read_bytes.sum.per_second", "pcie rd B/s (into GPU)"),
    ("pcie__write_bytes.sum.per_second", "pcie wr B/s (out of GPU)"),
    ("syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum", "sysmem rd sectors"),
    ("syslts__t_sectors_srcunit_tex_aperture_sysmem_op_write_lookup_miss.sum", "sysmem wr sectors"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-sb stall / issue"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[ix["Kernel Name"]].split("(")[0]
        a = agg.setdefault(k, [0, 0.0, r[ix["Grid Size"]]])
        a[0] += 1
        a[1] += float(r[ix["Metric Value"]]) * (1e-3 if r[ix["Metric Unit"]] == "ns" else 1.0)
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total µs | µs / launch | share | grid (last) |", "|---|---|---|---|---|---|"]
    for k, (n, us, g) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {us / n:.2f} | {us / tot:.1%} | {g} |")
    return out


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    cols = [(k, nm) for k, nm in KEYS if k in h]
    out = ["| kernel | " + " | ".join(f"{nm} [{u[h.index(k)]}]" for k, nm in cols) + " |",
           "|---|" + "---|" * len(cols)]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        out.append(f"| `{name}` | " + " | ".join(r[h.index(k)] for k, _ in cols) + " |")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--full", action="append", default=[])
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    for p in a.launches:
        lines += [f"## Launch list `{p}` (gpu__time_duration.sum, --clock-control none; cold, serialised)", ""]
        lines += launches(p) + [""]
    for p in a.full:
        lines += [f"## `ncu --set full` capture `{p}`", ""]
        lines += full(p) + [""]
    with open(a.out, "w") as f:
        f.write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
