"""One router per GPU, launched by tests/test_gpu_multi.py under torchrun
(world >= 2, NCCL).  Every rank scans its own shard of each slot, the routers
merge by the chosen exchange (dist.py: shard, push, pairs, bitmap, or the
literal all-reduce(max) of the stamps), reconstruct, and each rank checks its
reports -- and its cells, all of them or the ones it owns -- against the CPU
oracle's union-min merge of every shard (merge_rseas, snapshot.cpp:117-142;
pipeline.cpp:76-85), which each rank rebuilds from the same seeded shards.

    torchrun --nproc-per-node N tests/dist_worker.py --merge shard
Exit code 0 and "dist_worker ok" on rank 0 when every slot matched.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (test infrastructure: the checker)

GEO = dict(q=10, r=5, delta=8, eta=256)
K, THETA = 5, 128.0


def shard_pairs(seed, slot, rank):
    rng = O.Mt64(seed * 1000 + slot * 17 + rank)
    p = rng.pairs(20_000)
    # a super point split across the routers: each sees a third of its peers
    peers = O.Mt64(seed + slot).draw(300).astype(np.uint32)
    mine = peers[rank::3]
    sp = np.stack([np.full(mine.size, 0x0A0000AA, np.uint32), mine], 1)
    shared = O.Mt64(seed * 7 + slot).pairs(3000)  # pairs every router sees
    return np.concatenate([p, sp, shared])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--merge", default="shard", choices=["shard", "push", "pairs", "bitmap", "stamps"])
    ap.add_argument("--slots", type=int, default=4)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_1803_11036_b200 as P
    from paper_1803_11036_b200 import dist as PD

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    seed = 0x77
    shard = args.merge == "shard"
    g = P.Grid(seed=seed, device=local, k_max=K, shard=(world, rank) if shard else None, **GEO)
    g.set_stream(stream.cuda_stream)
    if args.merge != "stamps":
        ex = {"shard": PD.SHARD, "push": PD.PUSH, "pairs": PD.PAIRS, "bitmap": PD.BITMAP}[args.merge]
        PD.prepare(g, ex, region_cap=1 << 17)
    o = O.OracleGrid(seed=seed, **GEO)  # the union-min merged grid of every shard
    bad = 0
    for s in range(args.slots):
        mine = shard_pairs(seed, s, rank)
        g.scan_batch(torch.from_numpy(mine.view(np.int32)).cuda())
        for r in range(world):
            o.scan(shard_pairs(seed, s, r))
        if args.merge == "stamps":
            PD.merge_stamps_max(g)
        else:
            PD.merge(g)
        got = [(d.cip, d.estimate) for d in PD.reconstruct(g, K, THETA)]
        want = [(d.cip, d.estimate) for d in o.reconstruct(K, THETA)]
        lo, hi = g.owned()
        cells_ok = np.array_equal(g.cells_range(lo, hi - lo), o.cells()[lo:hi])
        if got != want or not cells_ok or 0x0A0000AA not in {c for c, _ in got}:
            bad += 1
            print(f"[rank {rank}] slot {s}: reports {'ok' if got == want else 'DIFFER'}, "
                  f"cells {'ok' if cells_ok else 'DIFFER'}", flush=True)
        g.advance_slot()
        o.advance()
    t = torch.tensor([bad], device=f"cuda:{local}")
    dist.all_reduce(t)
    if rank == 0:
        print("dist_worker ok" if int(t.item()) == 0 else f"dist_worker FAILED ({int(t.item())} rank-slots)",
              flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if int(t.item()) == 0 else 1)


if __name__ == "__main__":
    main()
