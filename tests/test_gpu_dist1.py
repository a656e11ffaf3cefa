"""The multi-router plumbing on the one GPU this box has: a 1-rank NCCL
group drives every exchange path of bench.py/dist.py end to end (symmetric
memory rendezvous and the peer table for PUSH, the all-gathers of PAIRS,
the OR all-reduce of BITMAP, the stamp all-reduce), so the calls and buffer
views are exercised on a real device; the algebra of 2- and 3-router
exchanges is covered by tests/test_dist_gloo.py."""
import socket

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DESK = dict(q=10, r=5, delta=8, eta=256)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def pg():
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["pairs", "push", "bitmap", "stamps", "shard"])
def test_exchange_paths_single_rank(gpu, pg, exchange):
    import torch

    from paper_1803_11036_b200 import dist as PD

    g = gpu.Grid(seed=0x44, **DESK)
    g.track_window(5)
    o = O.OracleGrid(seed=0x44, **DESK)
    if exchange != "stamps":
        PD.prepare(g, {"pairs": PD.PAIRS, "push": PD.PUSH, "bitmap": PD.BITMAP, "shard": PD.SHARD}[exchange],
                   region_cap=1 << 16)
    rng = O.Mt64(44)
    for s in range(3):
        p = rng.pairs(20_000)
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
        o.scan(p)
        if exchange == "stamps":
            PD.merge_stamps_max(g)
        else:
            PD.merge(g)
        assert np.array_equal(g.cells(), o.cells()), (exchange, s)
        assert [(d.cip, d.estimate) for d in PD.reconstruct(g, 5, 128.0)] == \
            [(d.cip, d.estimate) for d in o.reconstruct(5, 128.0)]
        g.advance_slot()
        o.advance()


@pytest.mark.parametrize("op", ["or", "and"])
def test_peer_bitwise_allreduce_single_rank(gpu, pg, op):
    """The peer-memory OR/AND all-reduce (symmetric staging buffer, device
    barriers, sspd_reduce_words over the peers' copies) on a 1-rank group:
    the reduce of one copy is the identity, over ragged lengths and a
    length past the staging buffer's first size."""
    import torch

    from paper_1803_11036_b200 import dist as PD

    for n in (1, 5, 1027, (1 << 20) + 13):
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda:0")
        want = x.clone()
        PD._bitwise_allreduce_peer_(x, op)
        torch.cuda.synchronize()
        assert torch.equal(x, want), n
