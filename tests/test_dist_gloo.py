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
    from paper_1803_11036_b200.dist import or_allreduce_

    g = torch.Generator().manual_seed(rank)
    for n in (1, 7, 64, 1001):  # padding paths
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, generator=g)
        parts = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(parts, x)
        want = parts[0].clone()
        for q in parts[1:]:
            want |= q
        or_allreduce_(x)
        if not torch.equal(x, want):
            out[rank] = False
            break
    else:
        out[rank] = True
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
