#!/usr/bin/env python
"""C4: window/slice sweep -- reconstruction cost versus scan cost for
k = 2..64 slices per window (BASELINE.json configs[3]).

Runs bench.py (device-resident C2 slots) once per window length and tabulates
the per-slot scan time, the reconstruction latency (fold + window counts +
hot sets + joins + finalize, reports on the host) and the reported hosts.
Stamp width: this build keeps u32 slice stamps only -- exact u16 distances
need >= 17 bits -- so the width axis of C4 is not swept.

    python tools/sweep_c4.py [--config c2] [--out profiles/r01_c4_window_sweep.md]
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
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for k in (2, 4, 8, 16, 32, 64):
        p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", args.config,
                            "--window", str(k), "--steps", "5", "--warmup", str(max(3, k)),
                            "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True)
        line = json.loads(p.stdout.strip().splitlines()[-1])
        share = line["kernels_share"]
        ms = line["ms_per_step"]
        rows.append((k, ms, share.get("scan", 0) * ms, line["reconstruct_ms"],
                     line["reports_last_step"], line["value"]))
        print(rows[-1], flush=True)
    out = ["| k (slots) | ms/slot | scan ms | reconstruct ms | reports | Mpkt/s |",
           "|---|---|---|---|---|---|"]
    out += [f"| {k} | {ms:.3f} | {sc:.3f} | {rc:.3f} | {n} | {v:.0f} |" for k, ms, sc, rc, n, v in rows]
    text = "\n".join(out) + "\n"
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(f"# C4 window sweep ({args.config}, B200, bench.py --window k)\n\n"
                    "Stamp width fixed at 32 bits (exactness of the u16 distance API needs >= 17).\n\n")
            f.write(text)


if __name__ == "__main__":
    main()
