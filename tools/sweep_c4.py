#!/usr/bin/env python
"""C4: window/slice sweep -- reconstruction cost versus scan cost for
k = 2..64 slices per window (BASELINE.json configs[3]).

Runs bench.py (device-resident C2 slots) once per (stamp width, window
length) and tabulates the per-slot scan time, the reconstruction latency
(window counts + hot sets + joins + finalize, reports on the host) and the
reported hosts.  Widths 8/16 are narrow-stamp grids (exact R_k for k up to
the window, plus the reports); 32 keeps full distances too.

    python tools/sweep_c4.py [--config c2] [--widths 8,16,32] [--out profiles/r01_c4_window_sweep.md]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--widths", default="8,16,32")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for w in [int(x) for x in args.widths.split(",")]:
        for k in (2, 4, 8, 16, 32, 64):
            p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", args.config,
                                "--window", str(k), "--stamp-width", str(w), "--steps", "5",
                                "--warmup", str(max(3, k)), "--no-cpu-baseline", "--no-e2e"],
                               capture_output=True, text=True)
            line = json.loads(p.stdout.strip().splitlines()[-1])
            share = line["kernels_share"]
            ms = line["ms_per_step"]
            acc = line["accuracy"]
            rows.append((w, k, ms, share.get("scan", 0) * ms, line["reconstruct_ms"],
                         line["reports_last_step"], acc.get("exact_fnr"), acc.get("exact_fpr"), line["value"]))
            print(rows[-1], flush=True)
    out = ["| stamp bits | k (slots) | grid GiB | ms/slot | scan ms | reconstruct ms | reports | FNR | FPR | Mpkt/s |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    cfg = {"c2": 5 * (1 << 16) * (1 << 16), "c1": 5 * (1 << 14) * 2048}.get(args.config, 0)
    out += [f"| {w} | {k} | {cfg * w / 8 / 2**30:.0f} | {ms:.3f} | {sc:.3f} | {rc:.3f} | {n} | {fn} | {fp} | {v:.0f} |"
            for w, k, ms, sc, rc, n, fn, fp, v in rows]
    text = "\n".join(out) + "\n"
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(f"# C4 window x stamp-width sweep ({args.config}, B200, "
                    "bench.py --window k --stamp-width w)\n\n"
                    "FNR/FPR against exact device counts of the window (sspd_exact_counts).\n\n")
            f.write(text)


if __name__ == "__main__":
    main()
