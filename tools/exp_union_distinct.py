"""Distinct (cip, oip) pairs in one C2 slot for 1 router vs the union over N
routers (the synth shards by j % N): how much merged work union-min adds."""
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
cdf = torch.from_numpy(B.zipf_cdf(L, cfg).view(np.int64)).cuda()
n = cfg["pairs_per_slot"]
for N in (1, 2, 4, 8):
    keys = []
    per = []
    for r in range(N):
        sp = B.synth_params(cfg, r, N)
        t = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        P._cabi.check(L.sspd_synth_device(0, C.byref(sp), C.c_void_p(cdf.data_ptr()), 0, 0, n,
                                          C.c_void_p(t.data_ptr()), None))
        k = (t[:, 0].to(torch.int64) << 32) | (t[:, 1].to(torch.int64) & 0xffffffff)
        u = torch.unique(k)
        per.append(u.numel())
        keys.append(u)
        del t, k
    total = torch.unique(torch.cat(keys)).numel()
    print(f"N={N}: distinct per router {np.mean(per) / 1e6:.2f}M, union {total / 1e6:.2f}M "
          f"({total / np.mean(per):.2f}x one router's)", flush=True)
    del keys
    torch.cuda.empty_cache()
