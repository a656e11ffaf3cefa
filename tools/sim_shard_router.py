"""One router's slot in an N-router ONE-HOP sharded deployment, timed on ONE
GPU (the relayed exchange's counterpart is tools/sim_relay_router.py).

The SHARD exchange (dist.py ShardExchange(relay=False)) cannot be timed here
with N GPUs, so this runs router 0's share of the work for real and produces
its inputs with helper grids: routers 1..N-1 scan their shards one after
another on the same device (pushing into router 0's inbox exactly as their
own GPUs would), then router 0 is timed on

  own scan (dedup, stamp owned cells, push new pairs to the other owners)
  + receive (the other routers' pushes: dedup against router 0's own keys,
    stamp owned cells; all regions in one launch, counts from device memory)
  + reconstruction (hot bits / masks merged in-process here; NCCL on N GPUs)

Collective / NVLink time is not included.  Round 2: every grid is PARTIAL (only
its cells, sspd_grid_create_sharded), so the full C2 geometry (eta 2^16) fits.

    python tools/sim_shard_router.py [--routers 8] [--eta 65536]
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
    ap.add_argument("--eta", type=int, default=1 << 16)
    args = ap.parse_args()
    N = args.routers
    cfg = dict(B.CONFIGS["c2"])
    cfg["eta"] = args.eta
    L = P.load()
    dev = 0
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cdf = torch.from_numpy(B.zipf_cdf(L, cfg).view(np.int64)).cuda()
    n = cfg["pairs_per_slot"]
    cap = 12 << 20  # pairs per (destination, source) region: a router's new pairs fit
    k, theta = cfg["k"], cfg["theta"]

    def shard(rank, slot, out):
        sp = B.synth_params(cfg, rank, N)
        P._cabi.check(L.sspd_synth_device(dev, C.byref(sp), C.c_void_p(cdf.data_ptr()), slot, 0, n,
                                          C.c_void_p(out.data_ptr()), C.c_void_p(stream.cuda_stream)))

    buf = torch.empty((n, 2), dtype=torch.int32, device="cuda")
    # router 0's inbox is read; routers 1..N-1's inboxes only receive (distinct buffers, as on N GPUs)
    inboxes = [torch.zeros(N * cap * 2, dtype=torch.int32, device="cuda") for _ in range(N)]
    table = torch.tensor([b.data_ptr() for b in inboxes], dtype=torch.int64, device="cuda")

    def grid(rank):
        g = P.Grid(cfg["q"], cfg["r"], cfg["delta"], cfg["seed"], cfg["eta"], device=dev, k_max=k,
                   shard=(N, rank) if N > 1 else None)
        g.set_stream(stream.cuda_stream)
        g.set_shard(table.data_ptr(), N, rank, cap)
        return g

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    r0 = grid(0)
    rows = []
    for slot in range(args.slots):
        # the other routers' scans, one at a time, pushing into router 0's inbox
        sent_to_0 = [0] * N
        for rank in range(1, N):
            h = grid(rank)  # a fresh pair set: it pushes exactly its slot's new pairs
            shard(rank, slot, buf)
            h.scan_device(buf.data_ptr(), n)
            h.synchronize()
            sent_to_0[rank] = PD.device_view(h.shard_sent_ptr(), 2 * N, dev).view(torch.int64)[0].item()
            h.close()
            del h
        shard(0, slot, buf)
        torch.cuda.synchronize()
        a = ev()
        r0.scan_device(buf.data_ptr(), n)
        b = ev()
        counts = torch.tensor(sent_to_0, dtype=torch.int64, device="cuda")
        r0.shard_receive_regions_dev(inboxes[0].data_ptr(), cap, counts.data_ptr(), 1, N, 0)
        c = ev()
        r0.shard_hot(k, theta)
        ns, mptr, words = r0.shard_select(k, theta)
        reps = r0.shard_finish(theta)
        d = ev()
        torch.cuda.synchronize()
        assert not r0.shard_overflow(), "a region ran past its capacity"
        own, recv, rec = a.elapsed_time(b), b.elapsed_time(c), c.elapsed_time(d)
        rows.append((slot, own, recv, rec, sum(sent_to_0)))
        r0.advance_slot()
        inboxes[0].zero_()
        print(f"slot {slot}: own {own:.3f} ms, receive {recv:.3f} ms ({sum(sent_to_0) / 1e6:.1f}M pairs), "
              f"reconstruct {rec:.3f} ms", file=sys.stderr, flush=True)
    rows = rows[1:]  # first slot: cold
    own = np.mean([r[1] for r in rows])
    recv = np.mean([r[2] for r in rows])
    rec = np.mean([r[3] for r in rows])
    got = np.mean([r[4] for r in rows]) / 1e6
    per_router = own + recv + rec
    print(f"# One router of {N} under the ONE-HOP SHARD exchange, partial grids, timed on one B200 "
          f"(`tools/sim_shard_router.py`)\n")
    print(f"C2 trace (1e8 Zipf pairs per router per slot), table q16 r5 delta6 eta {cfg['eta']}, k={k}; "
          f"mean of slots 1..{args.slots - 1}.\n")
    print("| phase | ms per slot |\n|---|---|")
    print(f"| own scan: dedup, stamp owned cells (1/{N} of them), push new pairs to owners | {own:.3f} |")
    print(f"| receive: dedup and stamp the {got:.1f}M pairs the other {N - 1} routers pushed here | {recv:.3f} |")
    print(f"| reconstruction on this router's hot bits (the merged sets are larger; collectives not included) "
          f"| {rec:.3f} |")
    print(f"| **router slot** | **{per_router:.3f}** |")
    print(f"\nPredicted aggregate at N={N} (no collective time): {N} x 1e8 / {per_router:.3f} ms = "
          f"{N * 1e8 / per_router / 1e6:.0f} Gpkt/s.")


if __name__ == "__main__":
    main()
