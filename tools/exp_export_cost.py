"""Scan time at C2 on one GPU with the exchange hooks on: plain dedup, EXPORT
(distinct-pair list, the PAIRS/PUSH exchanges) and SHARD (own scan with
pushes) at world 2/8 (pushes into local scratch inboxes)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
import paper_1803_11036_b200 as P  # noqa: E402

cfg = dict(B.CONFIGS["c2"])
cfg["eta"] = 1 << 15
L = P.load()
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
cdf = torch.from_numpy(B.zipf_cdf(L, cfg).view(np.int64)).cuda()
n = cfg["pairs_per_slot"]
buf = torch.empty((n, 2), dtype=torch.int32, device="cuda")
sp = B.synth_params(cfg, 0, 1)
P._cabi.check(L.sspd_synth_device(0, C.byref(sp), C.c_void_p(cdf.data_ptr()), 0, 0, n,
                                  C.c_void_p(buf.data_ptr()), C.c_void_p(stream.cuda_stream)))
cap = 24 << 20


def timed(g, reps=3):
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.scan_device(buf.data_ptr(), n)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        g.advance_slot()
    return sorted(ts)[len(ts) // 2]


for mode in ("dedup", "export", "shard2", "shard8"):
    g = P.Grid(cfg["q"], cfg["r"], cfg["delta"], cfg["seed"], cfg["eta"], k_max=cfg["k"])
    g.set_stream(stream.cuda_stream)
    keep = []
    if mode == "export":
        g.set_exchange(2)
    elif mode.startswith("shard"):
        w = int(mode[5:])
        boxes = [torch.zeros(w * cap * 2, dtype=torch.int32, device="cuda") for _ in range(w)]
        table = torch.tensor([b.data_ptr() for b in boxes], dtype=torch.int64, device="cuda")
        keep = [boxes, table]
        g.set_shard(table.data_ptr(), w, 0, cap)
    print(f"{mode}: scan {timed(g):.3f} ms", flush=True)
    g.close()
    del keep
    torch.cuda.empty_cache()
