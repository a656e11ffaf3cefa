"""Multi-router host logic on CPU: world_size 2 with gloo.

Each rank is a router with its own shard of every slot.  The union-min merge
of paper_1803_11036_b200/dist.py exchanges only the slot's touched bitmap
(OR all-reduce) and folds it into the rank's stamps.  Here the per-router
touches come from the CPU oracle and the fold is done on numpy stamps, so the
test checks the exchange and the stamp algebra end to end against the
reference semantics: every rank's grid must equal merge_rseas(node grids,
kUnionMin) of the oracle, and the single-node grid of the unsplit stream.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

GEO = dict(q=10, r=5, delta=8, seed=0x107, eta=256)
BASE_NOW = 65535


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def touched_bits(pairs):
    """The recorders a slot touches, as the device bitmap (LSB-first words)."""
    g = O.OracleGrid(**GEO)
    g.scan(pairs)
    bits = np.packbits(g.cells() == 0, bitorder="little")
    return np.frombuffer(bits.tobytes(), dtype=np.int32).copy()


def distances(stamps, now):
    age = (now - stamps.astype(np.int64))
    return np.minimum(age, 0xFFFF).astype(np.uint16)


def worker(rank, world, port, slots, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_11036_b200.dist import or_allreduce_

    rng = O.Mt64(1070)
    n_rec = GEO["r"] << GEO["q"]
    n_rec *= GEO["eta"]
    stamps = np.zeros(n_rec, dtype=np.uint32)
    now = BASE_NOW
    ok = True
    nodes = [O.OracleGrid(**GEO) for _ in range(world)]
    full = O.OracleGrid(**GEO)
    for s in range(slots):
        p = rng.pairs(3000)
        owner = rng.draw(3000) % world
        for i in range(world):
            nodes[i].scan(p[owner == i])
        full.scan(p)
        bits = torch.from_numpy(touched_bits(p[owner == rank]))
        or_allreduce_(bits)
        merged_bits = np.unpackbits(bits.numpy().view(np.uint8), bitorder="little")[:n_rec]
        stamps[merged_bits.astype(bool)] = now
        want = O.OracleGrid.merge(nodes, 0).cells()
        ok &= bool(np.array_equal(distances(stamps, now), want))
        ok &= bool(np.array_equal(distances(stamps, now), full.cells()))
        for n in nodes:
            n.advance()
        full.advance()
        now += 1
    out[rank] = ok
    dist.barrier()
    dist.destroy_process_group()


def test_union_min_exchange_two_routers():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(2, free_port(), 5, out), nprocs=2, join=True)
    assert out[0] and out[1]


def _or_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_11036_b200.dist import and_allreduce_, or_allreduce_

    g = torch.Generator().manual_seed(rank)
    ok = True
    for n in (1, 7, 64, 1001):  # padding paths
        for op, fn in (("or", or_allreduce_), ("and", and_allreduce_)):
            x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, generator=g)
            parts = [torch.empty_like(x) for _ in range(world)]
            dist.all_gather(parts, x)
            want = parts[0].clone()
            for q in parts[1:]:
                if op == "or":
                    want |= q
                else:
                    want &= q
            fn(x)
            ok = ok and torch.equal(x, want)
    out[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_or_allreduce(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_or_worker, args=(world, free_port(), out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))


def _pairs_worker(rank, world, port, slots, out):
    """The pair-list exchange: each router contributes its slot's distinct
    pairs; folding everyone's pairs gives the union-min merged grid."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_11036_b200.dist import exchange_pairs

    rng = O.Mt64(4242)
    mine = O.OracleGrid(**GEO)   # this router's merged view
    nodes = [O.OracleGrid(**GEO) for _ in range(world)]
    ok = True
    for s in range(slots):
        p = rng.pairs(2000)
        p = p[rng.draw(6000) % 2000]          # repeats, like Zipf traffic
        owner = rng.draw(len(p)) % world
        for i in range(world):
            nodes[i].scan(p[owner == i])
        local = np.unique(p[owner == rank], axis=0)   # the slot's distinct pairs
        mine.scan(local)
        for part in exchange_pairs(torch.from_numpy(local.view(np.int32).copy())):
            mine.scan(part.numpy().view(np.uint32))
        ok &= bool(np.array_equal(mine.cells(), O.OracleGrid.merge(nodes, 0).cells()))
        mine.advance()
        for n in nodes:
            n.advance()
    out[rank] = ok
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_pair_list_exchange(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_pairs_worker, args=(world, free_port(), 4, out), nprocs=world, join=True)
    assert all(out[r] for r in range(world))


def _shard_worker(rank, world, port, slots, out, relay=False):
    """The sharded union-min algebra (dist.py ShardExchange) on numpy grids:
    each router owns cells c with c * world // ncells == rank, stamps its own
    pairs' owned recorders, sends each pair to the owners of its other cells,
    stamps what it receives; hot bits are OR-merged and a host's bucket masks
    AND-merged.  Must equal the single merged grid: hot sets and every
    planted host's R_k."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1803_11036_b200.dist import and_allreduce_, or_allreduce_

    q, r, delta, eta, seed, k = 10, 5, 8, 256, 0x5a, 3
    ncells = r << q
    cutoff = O.hot_cutoff(eta, 128.0)
    stamps = np.zeros((ncells, eta), np.int64)      # this router's view (exact on owned cells)
    merged = np.zeros((ncells, eta), np.int64)      # the single merged grid, for reference
    owner = (np.arange(ncells) * world) // ncells
    cols_cache = {}

    def touches(cip, oip):
        if cip not in cols_cache:
            cols_cache[cip] = [(row << q) | c for row, c in enumerate(O.rhfg_cols(q, r, delta, seed, cip))]
        return cols_cache[cip], O.h1_raw(seed, oip) % eta

    ok = True
    now = 65535
    hosts = [0x0A000000 + h for h in range(3)]
    for slot in range(slots):
        rng = np.random.default_rng(1000 * slot + 7)
        everyone = []
        for src in range(world):  # every router's traffic, from a shared seed
            p = rng.integers(0, 2**32, size=(300, 2), dtype=np.uint64).astype(np.uint32)
            for h in hosts[: src + 1]:
                p = np.concatenate([p, np.stack([np.full(60, h, np.uint32),
                                                 rng.integers(0, 2**32, 60, dtype=np.uint64).astype(np.uint32)], 1)])
            everyone.append(p)
        for cip, oip in np.concatenate(everyone):
            cells, b = touches(int(cip), int(oip))
            merged[cells, b] = now
        own = everyone[rank]
        if relay:
            # hop 1: every new pair to its pair owner; the pair owner dedups
            # the union of what it got (its own share included)
            hop1 = [[] for _ in range(world)]
            for cip, oip in {(int(a), int(b)) for a, b in own}:
                hop1[hash((cip, oip)) % world].append((cip, oip))
            objs = [None] * world
            dist.all_gather_object(objs, hop1)
            own = sorted({pr for src in range(world) for pr in objs[src][rank]})
        outbox = [[] for _ in range(world)]
        for cip, oip in own:
            cells, b = touches(int(cip), int(oip))
            for c in cells:
                if owner[c] == rank:
                    stamps[c, b] = now
            for d in {int(owner[c]) for c in cells} - {rank}:  # once per owner (the kernel's dmask)
                outbox[d].append((int(cip), int(oip)))
        # the exchange: every router receives the pairs pushed (relayed) to it
        objs = [None] * world
        dist.all_gather_object(objs, outbox)
        received = [pr for src in range(world) if src != rank for pr in objs[src][rank]]
        if relay:  # each pair reaches a cell owner once, from its pair owner
            ok = ok and len(received) == len(set(received))
        for cip, oip in set(received):
            cells, b = touches(cip, oip)
            for c in cells:
                if owner[c] == rank:
                    stamps[c, b] = now
        mine = owner == rank
        ok = ok and np.array_equal(stamps[mine], merged[mine])
        # hot sets: per-owner R_k, OR-merged
        rk = ((stamps > 0) & (stamps > now - k)).sum(1)
        hot = torch.from_numpy(np.packbits((rk >= cutoff) & mine, bitorder="little").view(np.uint8).copy())
        hot32 = torch.zeros((hot.numel() + 3) // 4 * 4, dtype=torch.uint8)
        hot32[: hot.numel()] = hot
        hot32 = hot32.view(torch.int32)
        or_allreduce_(hot32)
        want = ((merged > 0) & (merged > now - k)).sum(1) >= cutoff
        got = np.unpackbits(hot32.view(torch.uint8).numpy(), bitorder="little")[:ncells].astype(bool)
        ok = ok and np.array_equal(got, want)
        # a host's R_k: AND over its r estimators, each router masking its owned rows
        for h in hosts:
            cells, _ = touches(h, 0)
            m = np.ones(eta, bool)
            for c in cells:
                if owner[c] == rank:
                    m &= (stamps[c] > 0) & (stamps[c] > now - k)
            words = torch.from_numpy(np.packbits(m, bitorder="little").view(np.int32).copy())
            and_allreduce_(words)
            got_rk = int(np.unpackbits(words.view(torch.uint8).numpy(), bitorder="little")[:eta].sum())
            want_rk = int(np.all([(merged[c] > 0) & (merged[c] > now - k) for c in cells], axis=0).sum())
            ok = ok and got_rk == want_rk
        now += 1
    out[rank] = ok
    dist.destroy_process_group()


@pytest.mark.parametrize("relay", [False, True], ids=["one_hop", "relayed"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_union_min_algebra(world, relay):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(world, free_port(), 4, out, relay), nprocs=world, join=True)
    assert all(out[r] for r in range(world))
