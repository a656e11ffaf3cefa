"""merge_rseas (snapshot.cpp:117-142) at the C1 geometry: n grids merged on
one B200 (sspd_merge: element-wise max/min of stamps) against the compiled
reference on the host cores (the C3 CPU row).

    python tools/bench_merge.py > profiles/r01_merge.md
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11036_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

GEO = dict(q=14, r=5, delta=6, eta=2048)
print(f"# merge_rseas at the C1 geometry (q14 r5 delta6 eta2048), {os.cpu_count()} host cores\n")
print("| n grids | policy | B200 ms (sspd_merge) | reference ms (merge_rseas) | speed-up |")
print("|---|---|---|---|---|")
for n in (2, 4, 8):
    rng = O.Mt64(n)
    gpu, ref = [], []
    for i in range(n):
        g = P.Grid(seed=0x5eed, **GEO)
        h = O.RefGrid(seed=0x5eed, **GEO)
        p = rng.pairs(1_000_000)
        g.scan_batch(p)
        h.scan(p, os.cpu_count())
        g.advance_slot()
        h.advance(os.cpu_count())
        gpu.append(g)
        ref.append(h)
    for policy, name in ((P.UNION_MIN, "union-min"), (P.PAPER_MAX, "paper-max")):
        out = P.merge_rseas(gpu, policy)
        out.synchronize()
        ts = []
        for _ in range(7):
            t0 = time.perf_counter()
            P.merge_rseas(gpu, policy, out=out)
            out.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        tg = sorted(ts)[3]
        tr = []
        for _ in range(3):
            t0 = time.perf_counter()
            m = O.RefGrid.merge(ref, policy)
            tr.append((time.perf_counter() - t0) * 1e3)
            del m
        tr = sorted(tr)[1]
        assert np.array_equal(out.cells(), O.RefGrid.merge(ref, policy).cells())
        print(f"| {n} | {name} | {tg:.2f} | {tr:.1f} | {tr / tg:.0f}x |", flush=True)
