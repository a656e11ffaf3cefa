"""Randomised differential tests: the CUDA path against the CPU oracle over
random valid geometries (validate_config's whole domain, hashing.cpp:63-87),
scan modes, stamp widths, windows and traffic mixes.  Seeded, so every run
checks the same cases; each case compares grids (32-bit), in-window counts,
hot sets and reconstruction reports -- or the CandidateOverflow level and
count -- slot by slot.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def random_geometry(rng):
    while True:
        q = int(rng.integers(2, 17))
        delta = int(rng.integers(1, q))
        r_min = max(3, -(-(32 - q) // delta) + 2)
        if r_min > 14:
            continue
        r = int(rng.integers(r_min, min(r_min + 3, 15) + 1))
        eta = int(rng.choice([2, 3, 7, 16, 40, 64, 100, 256, 1000]))
        if (r << q) * eta > (1 << 21):  # keep the oracle's per-slot work small
            continue
        return dict(q=q, r=r, delta=delta, eta=eta)


def recon_both(gpu, g, o, k, theta, cap):
    try:
        ref = o.reconstruct(k, theta, cap=cap)
    except O.CandidateOverflow as e:
        with pytest.raises(gpu.CandidateOverflow) as got:
            g.reconstruct_leveled(k, theta)
        return (got.value.level, got.value.count) == (e.level, e.count)
    got = g.reconstruct_leveled(k, theta)
    return [(d.cip, d.estimate) for d in got] == [(d.cip, d.estimate) for d in ref]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case", range(60))
def test_random_case(gpu, case):
    rng = np.random.default_rng(0xF0220 + case)
    geo = random_geometry(rng)
    seed = int(rng.integers(0, 2**63))
    width = int(rng.choice([32, 32, 16, 8]))
    k = int(rng.integers(1, 9))
    mode = int(rng.choice([-1, 0, 1, 2, 3]))
    g = gpu.Grid(seed=seed, width=width, k_max=k if width < 32 or rng.random() < 0.5 else 0, **geo)
    g.scan_mode(mode, int(rng.choice([-1, 0, 1])))
    cap = 1 << 18
    g.candidate_cap = cap
    o = O.OracleGrid(seed=seed, **geo)
    mt = O.Mt64(seed & 0xFFFFFFFF)
    theta = float(max(1.0, geo["eta"] * rng.uniform(0.2, 0.9)))
    hosts = [int(mt.next()) & 0xFFFFFFFF for _ in range(int(rng.integers(1, 5)))]
    for s in range(int(rng.integers(3, 7))):
        parts = [mt.pairs(int(rng.integers(0, 3000)))]
        for h in hosts:
            if rng.random() < 0.7:
                fan = int(rng.integers(1, 3 * geo["eta"] + 2))
                parts.append(np.stack([np.full(fan, h, np.uint32), mt.draw(fan).astype(np.uint32)], 1))
        p = np.concatenate(parts)
        if len(p) and rng.random() < 0.5:
            p = np.concatenate([p, p[: len(p) // 3]])  # repeats inside the slot
        g.scan_batch(p)
        o.scan(p)
        if width == 32:
            assert np.array_equal(g.cells(), o.cells()), (case, s)
        for kk in sorted({1, k}):
            assert np.array_equal(g.active_counts(kk), o.active_counts(kk)), (case, s, kk)
        hot = o.hot_sets(k, theta)
        assert [h.tolist() for h in g.hot_sets(k, theta)] == [h.tolist() for h in hot], (case, s)
        # the reference enumerates |H0|*|H1|*|H2| triples (rsea.cpp:184-200): only
        # compare reconstructions the oracle finishes quickly
        if int(np.prod([len(h) for h in hot[:3]], dtype=np.float64)) <= 20_000_000:
            assert recon_both(gpu, g, o, k, theta, cap), (case, s, geo, width, mode)
        adv = int(rng.choice([1, 1, 1, 2, 5]))
        g.advance_slot(slots=adv)
        for _ in range(adv):
            o.advance()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case", range(16))
def test_random_run_detection(gpu, case):
    """run_detection end to end (pipeline.cpp:16-89) against the oracle's: random
    geometry, shard count, merge policy, window (k, mu, start), traffic with
    planted super points, time-sorted shards scanned slot run by slot run."""
    rng = np.random.default_rng(0x5D37 + case)
    geo = random_geometry(rng)
    seed = int(rng.integers(0, 2**63))
    k = int(rng.integers(1, 7))
    mu = float(rng.choice([1.0, 2.0, 3.5]))
    start = int(rng.integers(0, 1000))
    theta = float(max(1.0, geo["eta"] * rng.uniform(0.3, 0.8)))
    n_shards = int(rng.integers(1, 5))
    policy = int(rng.integers(0, 2))
    mt = O.Mt64(seed & 0xFFFFFFFF)
    hosts = [int(mt.next()) & 0xFFFFFFFF for _ in range(int(rng.integers(1, 4)))]
    slots = int(rng.integers(2, 7))
    recs = []
    for s in range(slots):
        parts = [mt.pairs(int(rng.integers(0, 2000)))]
        for h in hosts:
            if rng.random() < 0.7:
                fan = int(rng.integers(1, 2 * geo["eta"] + 2))
                parts.append(np.stack([np.full(fan, h, np.uint32), mt.draw(fan).astype(np.uint32)], 1))
        p = np.concatenate(parts)
        p = p[rng.permutation(len(p))]
        ts = start + np.floor(s * mu + rng.uniform(0, mu, len(p)) * 0.999).astype(np.uint64)
        ts.sort()
        recs.append(np.concatenate([ts.astype(np.uint32)[:, None], p], 1))
    trace = np.concatenate(recs)
    owner = rng.integers(0, n_shards, len(trace))
    shards = [trace[owner == i] for i in range(n_shards)]  # each stays time sorted
    args = dict(q=geo["q"], r=geo["r"], delta=geo["delta"], seed=seed, eta=geo["eta"], mu=mu, k=k,
                start=start, theta=theta, policy=policy)
    try:
        n_slots, want = O.run_detection(shards, **args)
    except O.CandidateOverflow:
        with pytest.raises(gpu.CandidateOverflow):
            gpu.run_detection(shards, **args)
        return
    got = gpu.run_detection(shards, **args)
    assert len(got) == n_slots
    assert [(s, d.cip, d.estimate) for s, dets in got for d in dets] == \
           [(s, d.cip, d.estimate) for s, d in want], (case, geo, n_shards, policy, k, mu)


_SHARD_COMPARED = []  # (case, slot, reports) whose reconstructions were compared


@pytest.mark.timeout(300)
@pytest.mark.parametrize("case", range(12))
def test_random_sharded_routers(gpu, case):
    """Sharded routers on one device over random geometries (include/sspd_cuda.h
    "sharded routers"; dist.ShardExchange): world 2..5 partial grids, one or
    two hops, counts from the host or from device memory, hot bits / masks
    merged by sspd_reduce_words.  Every router's reports equal the oracle's
    union-min merge and its owned cells are bit-exact, every slot."""
    import torch

    from paper_1803_11036_b200 import dist as PD
    from paper_1803_11036_b200.grid import reduce_words

    rng = np.random.default_rng(0x5A4D + case)
    geo = random_geometry(rng)
    seed = int(rng.integers(0, 2**63))
    world = int(rng.integers(2, 6))
    relay = bool(rng.random() < 0.6)
    dev_counts = bool(rng.random() < 0.5)
    k = int(rng.integers(1, 7))
    theta = float(max(1.0, geo["eta"] * rng.uniform(0.5, 0.9)))
    cap = 1 << 16
    grids = [gpu.Grid(seed=seed, shard=(world, r), k_max=k, **geo) for r in range(world)]
    for g in grids:
        g.candidate_cap = 1 << 18
    in_a = [torch.zeros(world * cap * 2, dtype=torch.int32, device="cuda") for _ in range(world)]
    in_b = [torch.zeros(world * cap * 2, dtype=torch.int32, device="cuda") for _ in range(world)]
    ta = torch.tensor([b.data_ptr() for b in in_a], dtype=torch.int64, device="cuda")
    tb = torch.tensor([b.data_ptr() for b in in_b], dtype=torch.int64, device="cuda")
    for r, g in enumerate(grids):
        if relay:
            g.set_shard_relay(ta.data_ptr(), tb.data_ptr(), world, r, cap)
        else:
            g.set_shard(ta.data_ptr(), world, r, cap)
    o = O.OracleGrid(seed=seed, **geo)
    mt = O.Mt64(seed & 0xFFFFFFFF)
    hosts = [int(mt.next()) & 0xFFFFFFFF for _ in range(int(rng.integers(1, 4)))]

    def counts(hop):  # [src * world + dst] on the device, as the all-gather leaves them
        torch.cuda.synchronize()
        out = torch.cat([PD.device_view(g.shard_sent_ptr(), 128, 0).view(torch.int64)[32 * hop: 32 * hop + world]
                         for g in grids]).contiguous()
        torch.cuda.synchronize()
        return out

    def receive(boxes, hop):
        sent = counts(hop)
        host = sent.view(world, world).tolist()
        for dst, g in enumerate(grids):
            if dev_counts:
                g.shard_receive_regions_dev(boxes[dst].data_ptr(), cap, sent.data_ptr() + 8 * dst, world, world, dst)
            else:
                box = boxes[dst].view(world, cap, 2)
                for src in range(world):
                    if src != dst and host[src][dst]:
                        g.shard_receive(box[src].data_ptr(), host[src][dst])

    for s in range(int(rng.integers(2, 5))):
        shared = mt.pairs(int(rng.integers(0, 300)))
        for r, g in enumerate(grids):
            parts = [mt.pairs(int(rng.integers(0, 600))), shared]
            for h in hosts:
                if rng.random() < 0.6:
                    fan = int(rng.integers(1, geo["eta"] + 2))
                    parts.append(np.stack([np.full(fan, h, np.uint32), mt.draw(fan).astype(np.uint32)], 1))
            p = np.concatenate(parts)
            if len(p):
                g.scan_batch(torch.from_numpy(np.ascontiguousarray(p).view(np.int32)).cuda())
            o.scan(p)
        if relay:
            sent = counts(0)
            for po, g in enumerate(grids):
                if dev_counts:
                    g.shard_relay_regions_dev(in_a[po].data_ptr(), cap, sent.data_ptr() + 8 * po, world, world)
                else:
                    g.shard_relay_regions(in_a[po].data_ptr(), cap, sent.view(world, world)[:, po].tolist())
            receive(in_b, 1)
        else:
            receive(in_a, 0)
        torch.cuda.synchronize()
        assert not any(g.shard_overflow() for g in grids)
        hot = [g.shard_hot(k, theta) for g in grids]
        merged = torch.empty(hot[0][1], dtype=torch.int32, device="cuda")
        reduce_words(0, [p for p, _ in hot], hot[0][1], "or", merged.data_ptr())
        torch.cuda.synchronize()
        for p, _ in hot:
            reduce_words(0, [merged.data_ptr()], hot[0][1], "or", p)
        torch.cuda.synchronize()
        cells = o.cells()
        for g in grids:
            lo, hi = g.owned()
            assert np.array_equal(g.cells_range(lo, hi - lo), cells[lo:hi]), (case, s)
        # only reconstructions the oracle's triple enumeration finishes quickly
        hot_o = o.hot_sets(k, theta)
        if int(np.prod([len(h) for h in hot_o[:3]], dtype=np.float64)) > 20_000_000:
            for g in grids:
                g.advance_slot()
            o.advance()
            continue
        try:
            want = o.reconstruct(k, theta, cap=1 << 18)
        except O.CandidateOverflow as e:
            with pytest.raises(gpu.CandidateOverflow) as got:
                grids[0].shard_select(k, theta)
            assert (got.value.level, got.value.count) == (e.level, e.count)
            return
        sel = [g.shard_select(k, theta) for g in grids]
        if sel[0][0]:
            w = sel[0][2]
            anded = torch.empty(w, dtype=torch.int32, device="cuda")
            reduce_words(0, [p for _, p, _ in sel], w, "and", anded.data_ptr())
            torch.cuda.synchronize()
            for _, p, _ in sel:
                reduce_words(0, [anded.data_ptr()], w, "and", p)
            torch.cuda.synchronize()
        for g in grids:
            assert [(d.cip, d.estimate) for d in g.shard_finish(theta)] == \
                [(d.cip, d.estimate) for d in want], (case, s, geo, world, relay, dev_counts)
        _SHARD_COMPARED.append((case, s, len(want)))
        for g in grids:
            g.advance_slot()
        o.advance()


def test_random_sharded_routers_compared_reports(gpu):
    """The sharded fuzz cases above must have compared real reconstructions
    (slots whose hot sets the oracle enumerates quickly), some with reports."""
    if not _SHARD_COMPARED:
        pytest.skip("run with the sharded fuzz cases")
    assert len(_SHARD_COMPARED) >= 12 and sum(1 for *_, n in _SHARD_COMPARED if n) >= 3, _SHARD_COMPARED
