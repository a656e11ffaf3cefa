"""Where a grid's lifetime goes: create, first scan, hot_sets, destroy (host
wall clock, paper geometry q14 r5 delta6 eta2048, ring k=5)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11036_b200 as P  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    pairs = rng.integers(0, 2**32, size=(1 << 20, 2), dtype=np.uint64).astype(np.uint32)
    for it in range(4):
        t = [time.perf_counter()]
        g = P.Grid(14, 5, 6, 0x5EED, 2048, k_max=5)
        t.append(time.perf_counter())
        g.scan_batch(pairs)
        g.synchronize()
        t.append(time.perf_counter())
        g.scan_batch(pairs)
        g.synchronize()
        t.append(time.perf_counter())
        g.hot_sets(5, 1024.0)
        t.append(time.perf_counter())
        g.close()
        t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        print(f"iter {it}: create {d[0]:.1f} ms, first scan {d[1]:.1f}, second scan {d[2]:.1f}, hot_sets {d[3]:.1f}, "
              f"destroy {d[4]:.1f}", flush=True)


if __name__ == "__main__":
    main()
