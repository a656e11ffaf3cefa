"""Reconstruction latency at C1 and C2 geometry: wall time per call (Python
and raw C ABI), device time of the queued kernels, and the gap between them."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11036_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

for name, geo, k, theta in [("C1", dict(q=14, r=5, delta=6, eta=2048), 5, 1024.0),
                            ("C2 geometry", dict(q=16, r=5, delta=6, eta=1 << 16), 5, 1024.0)]:
    g = P.Grid(seed=0x5eed, **geo)
    g.track_window(k)
    rng = O.Mt64(3)
    for s in range(3):
        for h in range(20):
            cip = int(rng.next()) & 0xffffffff
            fan = int(2 * theta)
            g.scan_batch(np.stack([np.full(fan, cip, np.uint32), rng.draw(fan).astype(np.uint32)], 1))
        g.scan_batch(rng.pairs(1_000_000))
        g.advance_slot()
    for _ in range(20):
        g.reconstruct_leveled(k, theta)
    g.synchronize()
    reps = 200
    t0 = time.perf_counter()
    for _ in range(reps):
        d = g.reconstruct_leveled(k, theta)
    t_py = (time.perf_counter() - t0) / reps * 1e3
    L = P.load()
    buf = (P._cabi.Detection_t * 4096)()
    n, lvl, cnt = C.c_uint64(), C.c_uint32(), C.c_uint64()
    cut = P.hot_cutoff(geo["eta"], theta)
    t0 = time.perf_counter()
    for _ in range(reps):
        L.sspd_reconstruct(g._h, k, cut, 1 << 24, buf, 4096, C.byref(n), C.byref(lvl), C.byref(cnt))
    t_c = (time.perf_counter() - t0) / reps * 1e3
    g.profile(True)
    g.profile_reset()
    for _ in range(reps):
        L.sspd_reconstruct(g._h, k, cut, 1 << 24, buf, 4096, C.byref(n), C.byref(lvl), C.byref(cnt))
    dev = 0.0
    for kn in ("reconstruct",):  # one event pair around the launch chain
        t, c, _ = g.profile_read(kn)
        dev += t
    g.profile(False)
    print(f"{name}: {len(d)} reports; per call: python {t_py:.3f} ms, C ABI {t_c:.3f} ms, "
          f"device (queued chain incl. read-back) {dev / reps:.3f} ms", flush=True)
