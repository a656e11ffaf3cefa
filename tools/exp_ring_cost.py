"""Scan-kernel time at C2 with and without the window ring (track_window):
what the ring's atomics cost inside scan_dedup_kernel."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
import paper_1803_11036_b200 as P  # noqa: E402

cfg = B.CONFIGS["c2"]
L = P.load()
dev = 0
torch.cuda.set_device(dev)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
cdf = torch.from_numpy(B.zipf_cdf(L, cfg).view(np.int64)).cuda()
sp = B.synth_params(cfg, 0, 1)
n = cfg["pairs_per_slot"]
trace = torch.empty((4, n, 2), dtype=torch.int32, device="cuda")
for s in range(4):
    P._cabi.check(L.sspd_synth_device(dev, C.byref(sp), C.c_void_p(cdf.data_ptr()), s, 0, n,
                                      C.c_void_p(trace[s].data_ptr()), C.c_void_p(stream.cuda_stream)))
torch.cuda.synchronize()
for ring in (5, 0):
    g = P.Grid(cfg["q"], cfg["r"], cfg["delta"], cfg["seed"], cfg["eta"], device=dev)
    g.set_stream(stream.cuda_stream)
    if ring:
        g.track_window(ring)
    for i in range(3):
        g.scan_device(trace[i % 4].data_ptr(), n)
        g.advance_slot()
    g.profile(True)
    g.profile_reset()
    for i in range(6):
        g.scan_device(trace[(i + 3) % 4].data_ptr(), n)
        g.advance_slot()
    t, k, _ = g.profile_read("scan")
    print(f"ring K={ring}: scan {t / k:.3f} ms/slot over {k} launches", flush=True)
    g.profile(False)
    g.close()
    torch.cuda.synchronize()
