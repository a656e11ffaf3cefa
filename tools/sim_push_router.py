"""One router's slot under the replicated exchanges (PAIRS / PUSH: every
router keeps the whole merged table), timed on ONE GPU -- the counterpart of
tools/sim_shard_router.py.  Routers 1..N-1 scan their shards one after
another on the same device and leave their new-pair lists; router 0 is timed
on its own scan (with the list export) plus scanning the other routers' lists
plus reconstruction.  Collective / NVLink time is not included.

    python tools/sim_push_router.py [--routers 8]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
import paper_1803_11036_b200 as P  # noqa: E402
from paper_1803_11036_b200 import dist as PD  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--routers", type=int, default=8)
    ap.add_argument("--slots", type=int, default=4)
    args = ap.parse_args()
    N = args.routers
    cfg = dict(B.CONFIGS["c2"])
    cfg["eta"] = 1 << 15
    L = P.load()
    dev = 0
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cdf = torch.from_numpy(B.zipf_cdf(L, cfg).view(np.int64)).cuda()
    n = cfg["pairs_per_slot"]
    k, theta = cfg["k"], cfg["theta"]
    buf = torch.empty((n, 2), dtype=torch.int32, device="cuda")

    def shard(rank, slot):
        sp = B.synth_params(cfg, rank, N)
        P._cabi.check(L.sspd_synth_device(dev, C.byref(sp), C.c_void_p(cdf.data_ptr()), slot, 0, n,
                                          C.c_void_p(buf.data_ptr()), C.c_void_p(stream.cuda_stream)))

    def grid():
        g = P.Grid(cfg["q"], cfg["r"], cfg["delta"], cfg["seed"], cfg["eta"], device=dev, k_max=k)
        g.set_stream(stream.cuda_stream)
        g.set_exchange(2)
        return g

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    r0 = grid()
    rows = []
    for slot in range(args.slots):
        lists = []
        for rank in range(1, N):
            h = grid()
            shard(rank, slot)
            h.scan_device(buf.data_ptr(), n)
            h.synchronize()
            ptr, cnt = h.new_pairs_ptr()
            lists.append(PD.device_view(ptr, 2 * cnt, dev).clone())
            h.close()
            del h
        shard(0, slot)
        torch.cuda.synchronize()
        a = ev()
        r0.scan_device(buf.data_ptr(), n)
        b = ev()
        r0.set_exchange(0)  # received lists are not re-exported
        for lst in lists:
            r0.scan_device(lst.data_ptr(), lst.numel() // 2)
        r0.set_exchange(2)
        c = ev()
        r0.reconstruct_leveled(k, theta)
        d = ev()
        torch.cuda.synchronize()
        got = sum(x.numel() // 2 for x in lists)
        rows.append((a.elapsed_time(b), b.elapsed_time(c), c.elapsed_time(d), got))
        print(f"slot {slot}: own {rows[-1][0]:.3f} ms, receive {rows[-1][1]:.3f} ms ({got / 1e6:.1f}M pairs), "
              f"reconstruct {rows[-1][2]:.3f} ms", file=sys.stderr, flush=True)
        r0.advance_slot()
        del lists
    rows = rows[1:]
    own, recv, rec = (np.mean([r[i] for r in rows]) for i in range(3))
    got = np.mean([r[3] for r in rows]) / 1e6
    per = own + recv + rec
    print(f"# One router of {N} under the replicated PAIRS/PUSH exchange, timed on one B200 "
          f"(`tools/sim_push_router.py`)\n")
    print("| phase | ms per slot |\n|---|---|")
    print(f"| own scan with the new-pair list export | {own:.3f} |")
    print(f"| receive: scan the {got:.1f}M pairs of the other {N - 1} routers' lists into the whole table | {recv:.3f} |")
    print(f"| reconstruction | {rec:.3f} |")
    print(f"| **router slot** | **{per:.3f}** |")
    print(f"\nPredicted aggregate at N={N} (no collective time): {N * 1e8 / per / 1e6:.0f} Gpkt/s.")


if __name__ == "__main__":
    main()
