#!/usr/bin/env python
"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launches.csv>      # per-kernel share of a launch list
  python tools/ncu_summary.py full <report.ncu-rep>        # key counters per profiled kernel
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "lts__t_sector_op_read_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "lts__t_requests_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = {}
    unit = None
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"^void ", "", r[ki].split("(")[0])
        tot.setdefault(name, [0.0, 0])
        tot[name][0] += float(r[vi].replace(",", ""))
        tot[name][1] += 1
        unit = r[ui]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
    total = sum(v for v, _ in tot.values())
    print("| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|")
    for name, (v, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
        print(f"| `{name}` | {c} | {v * scale:.3f} | {v * scale / c:.4f} | {v / total:.3f} |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"### `{r[hdr.index('Kernel Name')][:90]}`\n")
        print("| metric | unit | value |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {k} | {units[i]} | {r[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
