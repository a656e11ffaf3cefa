"""One router's slot under the RELAYED shard exchange (two hops), timed on
ONE GPU -- the counterpart of tools/sim_shard_router.py.  All routers' hops
run on the same device in lockstep (helper grids for routers 1..N-1, one at a
time); router 0 is timed on

  own scan (dedup; each new pair pushed to its pair owner; no stamping)
  + relay (dedup its share of the routers' union; stamp own cells; push once
    to each other cell owner)
  + receive (stamp what the pair owners relayed to it)
  + reconstruction on its own hot bits.

Collective / NVLink time is not included.  Round 2: every router's grid is
PARTIAL (only its cells, sspd_grid_create_sharded), so the full C2 geometry
(eta 2^16) fits -- router 0 plus one helper at a time -- and router 0's relay
and receive take their counts from device memory in one launch each
(sspd_shard_relay_regions_dev / sspd_shard_receive_regions_dev), as
dist.ShardExchange runs them.

    python tools/sim_relay_router.py [--routers 8] [--eta 65536]
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
    k, theta = cfg["k"], cfg["theta"]
    cap = (24 << 20) // N + (4 << 20)  # per (destination, source) region
    buf = torch.empty((n, 2), dtype=torch.int32, device="cuda")
    in_a = [torch.zeros(N * cap * 2, dtype=torch.int32, device="cuda") for _ in range(N)]
    in_b = [torch.zeros(N * cap * 2, dtype=torch.int32, device="cuda") for _ in range(N)]
    ta = torch.tensor([b.data_ptr() for b in in_a], dtype=torch.int64, device="cuda")
    tb = torch.tensor([b.data_ptr() for b in in_b], dtype=torch.int64, device="cuda")

    def shard(rank, slot):
        sp = B.synth_params(cfg, rank, N)
        P._cabi.check(L.sspd_synth_device(dev, C.byref(sp), C.c_void_p(cdf.data_ptr()), slot, 0, n,
                                          C.c_void_p(buf.data_ptr()), C.c_void_p(stream.cuda_stream)))

    def grid(rank):
        g = P.Grid(cfg["q"], cfg["r"], cfg["delta"], cfg["seed"], cfg["eta"], device=dev, k_max=k,
                   shard=(N, rank) if N > 1 else None)
        g.set_stream(stream.cuda_stream)
        g.set_shard_relay(ta.data_ptr(), tb.data_ptr(), N, rank, cap)
        return g

    def sent(g):
        g.synchronize()
        return PD.device_view(g.shard_sent_ptr(), 128, dev).view(torch.int64).tolist()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    r0 = grid(0)
    rows = []
    for slot in range(args.slots):
        for b in in_a + in_b:
            b.zero_()
        sa = [None] * N
        # hop 1 of routers 1..N-1 (fresh helpers: their pair sets start empty, as each slot's do)
        for rank in range(1, N):
            h = grid(rank)
            shard(rank, slot)
            h.scan_device(buf.data_ptr(), n)
            sa[rank] = sent(h)
            h.close()
            del h
        shard(0, slot)
        torch.cuda.synchronize()
        t0 = ev()
        r0.scan_device(buf.data_ptr(), n)
        t1 = ev()
        sa[0] = sent(r0)
        # hop 2: the other pair owners relay (helpers), then router 0 relays (timed)
        sb = [None] * N
        for po in range(1, N):
            h = grid(po)
            h.shard_relay_regions(in_a[po].data_ptr(), cap, [sa[src][po] for src in range(N)])
            sb[po] = sent(h)
            h.close()
            del h
        counts_a = torch.tensor([sa[src][0] for src in range(N)], dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        t2 = ev()
        r0.shard_relay_regions_dev(in_a[0].data_ptr(), cap, counts_a.data_ptr(), 1, N)
        t3 = ev()
        sb[0] = sent(r0)
        got = sum(sb[src][32] for src in range(1, N))
        counts_b = torch.tensor([sb[src][32] for src in range(N)], dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        t4 = ev()
        r0.shard_receive_regions_dev(in_b[0].data_ptr(), cap, counts_b.data_ptr(), 1, N, 0)
        t5 = ev()
        r0.shard_hot(k, theta)
        r0.shard_select(k, theta)
        r0.shard_finish(theta)
        t6 = ev()
        torch.cuda.synchronize()
        assert not r0.shard_overflow(), "a region ran past its capacity"
        relay_in = sum(sa[src][0] for src in range(N))
        rows.append((t0.elapsed_time(t1), t2.elapsed_time(t3), t4.elapsed_time(t5), t5.elapsed_time(t6), relay_in, got))
        print(f"slot {slot}: own {rows[-1][0]:.3f} ms, relay {rows[-1][1]:.3f} ms ({relay_in / 1e6:.1f}M in), receive "
              f"{rows[-1][2]:.3f} ms ({got / 1e6:.1f}M), reconstruct {rows[-1][3]:.3f} ms", file=sys.stderr, flush=True)
        r0.advance_slot()
    rows = rows[1:]
    own, relay, recv, rec = (np.mean([r[i] for r in rows]) for i in range(4))
    rin, got = (np.mean([r[i] for r in rows]) / 1e6 for i in (4, 5))
    per = own + relay + recv + rec
    print(f"# One router of {N} under the RELAYED shard exchange (two hops), partial grids, device-counted "
          f"relay/receive, eta {cfg['eta']}, timed on one B200 (`tools/sim_relay_router.py`)\n")
    print("| phase | ms per slot |\n|---|---|")
    print(f"| own scan: dedup, push each new pair to its pair owner (no stamping) | {own:.3f} |")
    print(f"| relay: dedup the {rin:.1f}M pairs routed to this pair owner, stamp own cells, push once per owner "
          f"| {relay:.3f} |")
    print(f"| receive: stamp the {got:.1f}M pairs relayed here | {recv:.3f} |")
    print(f"| reconstruction on this router's hot bits (collectives not included) | {rec:.3f} |")
    print(f"| **router slot** | **{per:.3f}** |")
    print(f"\nPredicted aggregate at N={N} (no collective time): {N * 1e8 / per / 1e6:.0f} Gpkt/s.")


if __name__ == "__main__":
    main()
