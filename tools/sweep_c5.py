#!/usr/bin/env python
"""C5: threshold and table-size sweep measuring detection accuracy (FPR/FNR
against exact ground truth) -- BASELINE.json configs[4], SURVEY.md §8d.

Runs the reference workflow through this repository's `sspd` CLI:
synth (planted bands at 0.5/0.8/1.0/1.2/2/4 x theta over Zipf background)
-> oracle (exact sliding-window counts) -> detect (B200) -> eval.  Prints a
markdown table; FPR/FNR are normalised by the true super points as in the
reference's evaluate (workload.cpp:360-385).

    python tools/sweep_c5.py [--out profiles/r01_c5_accuracy.md]
"""
import argparse
import os
import subprocess
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SSPD = os.path.join(ROOT, "paper_1803_11036_b200", "bin", "sspd")


def sh(*args):
    p = subprocess.run([SSPD, *map(str, args)], capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"{args[0]} failed ({p.returncode}): {p.stderr}")
    return p.stdout


def spec_text(theta, slots=20):
    lines = [f"slots {slots}",
             "background hosts=20000 zipf=1.1 pairs-per-slot=20000 max-distinct=64"]
    ip = 0x0A000000
    for mult, n in ((0.5, 10), (0.8, 10), (1.0, 4), (1.2, 10), (2.0, 10), (4.0, 4)):
        for _ in range(n):
            a = f"{ip >> 24}.{ip >> 16 & 255}.{ip >> 8 & 255}.{ip & 255}"
            lines.append(f"super cip={a} count={int(mult * theta)} from=0 to={slots - 1}")
            ip += 997
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--k", type=int, default=10)
    args = ap.parse_args()
    rows = []
    grid = [(theta, eta, q) for theta in (256, 512, 1024, 2048, 4096)
            for eta in (1 << 9, 1 << 11, 1 << 13) for q in (12, 14, 16)]
    with tempfile.TemporaryDirectory() as tmp:
        for theta, eta, q in grid:
            delta = 7 if q == 12 else 6  # coverage (r-2)*delta+q >= 32
            spec = os.path.join(tmp, "spec.txt")
            open(spec, "w").write(spec_text(theta))
            trace = os.path.join(tmp, "t.bin")
            truth = os.path.join(tmp, "truth.csv")
            rep = os.path.join(tmp, "rep.csv")
            ev = os.path.join(tmp, "eval.csv")
            common = ["--k", args.k, "--seed", "c5", "--eta", eta, "--q", q, "--r", 5,
                      "--delta", delta, "--theta", theta]
            sh("synth", spec, *common, "-o", trace, "--truth-out", truth)
            t0 = time.time()
            sh("detect", trace, *common, "-o", rep)
            dt = time.time() - t0
            sh("eval", "--reports", rep, "--truth", truth, "--theta", theta, "-o", ev)
            mean = [line for line in open(ev) if line.startswith("mean,")][0].strip().split(",")
            rows.append((theta, eta, q, float(mean[1]), float(mean[2]), float(mean[3]), dt))
            print(rows[-1], flush=True)
    out = ["| theta | eta | q | mean FPR | mean FNR | mean TFR | detect wall s |",
           "|---|---|---|---|---|---|---|"]
    out += [f"| {t} | {e} | {q} | {fp:.4f} | {fn:.4f} | {tf:.4f} | {dt:.2f} |"
            for t, e, q, fp, fn, tf, dt in rows]
    text = "\n".join(out) + "\n"
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write("# C5 accuracy sweep (B200, sspd CLI; exact truth from `sspd oracle`)\n\n")
            f.write(f"k={args.k} slots, 20 slots, Zipf background 20000 hosts x 20000 pairs/slot "
                    "(<=64 distinct each), planted bands at 0.5/0.8/1.0/1.2/2/4 x theta.\n\n")
            f.write(text)


if __name__ == "__main__":
    main()
