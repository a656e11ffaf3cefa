"""The compact key set of the pipelined dedup scan (kernels.cuh
scan_cset_kernel) against the CPU oracle.

The set keys a pair by (cip, bucket(oip)) and stores a 48-bit permutation of
the key as home slot + remainder, so a match must be exact (a false "seen"
would lose a touch) and a repeat must be found (the fresh-key device counter
equals the number of distinct keys).  Grids, in-window counts and the set's
own count are compared with the oracle / numpy over repeated, bucket-colliding
and table-overflowing traffic, with the set on and off.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DESK = dict(q=10, r=5, delta=8, eta=256)
PAPER = dict(q=14, r=5, delta=6, eta=2048)
ODD = dict(q=12, r=7, delta=4, eta=1000)
WIDE = dict(q=16, r=8, delta=6, eta=64)
E16 = dict(q=12, r=5, delta=7, eta=65536)   # the largest eta the set takes (48-bit keys)


def _grid(gpu, geo, seed, cset, k=4, passes=1):
    env = {"SSPD_CSET": "1" if cset else "0", "SSPD_CSET_PASSES": str(passes)}
    old = {key: os.environ.get(key) for key in env}
    os.environ.update(env)
    try:
        g = gpu.Grid(seed=seed, **geo)
    finally:
        for key, v in old.items():
            if v is None:
                del os.environ[key]
            else:
                os.environ[key] = v
    g.scan_mode(2, -1)
    g.track_window(k)
    return g


def bucket_fn(seed, eta):
    """Vectorised hash_opposite (hashing.hpp:56-59) from h1_raw: h1 is the XOR
    of four byte tables, so h1(x) = U0[b0]^U1[b1]^U2[b2]^U3[b3]^h1(0) with
    Ui[b] = h1(b << 8i)."""
    z = O.h1_raw(seed, 0)
    U = np.array([[O.h1_raw(seed, b << (8 * i)) for b in range(256)] for i in range(4)], dtype=np.uint64)

    def f(oip):
        oip = oip.astype(np.uint64)
        h = np.full(oip.shape, z, dtype=np.uint64)
        for i in range(4):
            h ^= U[i][(oip >> np.uint64(8 * i)) & np.uint64(0xFF)]
        return (h % np.uint64(eta)).astype(np.uint64)
    return f


def distinct_keys(pairs, bucket):
    keys = (pairs[:, 0].astype(np.uint64) << np.uint64(16)) | bucket(pairs[:, 1])
    return len(np.unique(keys))


def colliding_traffic(rng, seed, eta, hosts, per_host, n):
    """Each host sends to many oips, several of which share a bucket: the set
    must dedup them as one key, and keep hosts apart."""
    cips = rng.draw(hosts).astype(np.uint32)
    oips = rng.draw(hosts * per_host).astype(np.uint32).reshape(hosts, per_host)
    pick_h = rng.draw(n) % hosts
    pick_o = rng.draw(n) % per_host
    return np.stack([cips[pick_h], oips[pick_h, pick_o]], 1).astype(np.uint32)


@pytest.mark.parametrize("cset", [(1, 1), (1, 2), (1, 4), (0, 1)], ids=["keyset", "keyset_2pass", "keyset_4pass",
                                                                    "pairset"])
@pytest.mark.parametrize("geo", [DESK, PAPER, ODD, WIDE, E16], ids=["desk", "paper", "odd_eta", "wide_r", "eta65536"])
def test_keyset_scan_bit_exact(gpu, geo, cset):
    g = _grid(gpu, geo, 0x5eed, cset[0], passes=cset[1])
    o = O.OracleGrid(seed=0x5eed, **geo)
    rng = O.Mt64(11)
    for s in range(4):
        p = colliding_traffic(rng, 0x5eed, geo["eta"], 2000, 3 * geo["eta"] // 2 + 1, 120_000)
        u = rng.pairs(30_000)
        for part in (p[:70_000], u, p[70_000:], p[:20_000]):
            g.scan_batch(part)
            o.scan(part)
        assert np.array_equal(g.cells(), o.cells()), s
        assert np.array_equal(g.active_counts(3), o.active_counts(3)), s
        g.advance_slot()
        o.advance()


@pytest.mark.parametrize("passes", [1, 2])
@pytest.mark.parametrize("geo", [DESK, PAPER, E16], ids=["desk", "paper", "eta65536"])
def test_keyset_counts_distinct_keys(gpu, geo, passes):
    """The fresh-key counter equals the distinct (cip, bucket) keys of each
    slot: no repeat is missed and no new key is taken for a seen one."""
    g = _grid(gpu, geo, 0x1234, 1, passes=passes)
    bucket = bucket_fn(0x1234, geo["eta"])
    rng = O.Mt64(5)
    for s in range(3):
        p = colliding_traffic(rng, 0x1234, geo["eta"], 5000, 40, 400_000)
        before = g.fresh_pairs()
        g.scan_batch(p[:250_000])
        g.scan_batch(p[250_000:])
        assert g.fresh_pairs() - before == distinct_keys(p, bucket), s
        g.advance_slot()


@pytest.mark.slow
def test_keyset_overfull_table(gpu):
    """More distinct keys than the 2^24-entry table holds: probes hit the
    limit and read as fresh (redundant stamps only); the grid stays exact."""
    import torch

    geo = DESK
    g = _grid(gpu, geo, 0x77, 1, k=3)
    o = O.OracleGrid(seed=0x77, **geo)
    rng = O.Mt64(1)
    for s in range(2):
        p = rng.pairs(20_000_000)
        p[1::7] = p[::7][: len(p[1::7])]  # some repeats among the overflow
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
        o.scan(p)
        assert np.array_equal(g.cells(), o.cells()), s
        assert np.array_equal(g.active_counts(3), o.active_counts(3)), s
        g.advance_slot()
        o.advance()


def test_keyset_survives_cells_writes_and_slot_reset(gpu):
    """A cells() write inside a slot clears the set (its skips would be
    stale); advancing clears it too, so a pair seen last slot stamps again."""
    g = _grid(gpu, DESK, 0x31, 1)
    o = O.OracleGrid(seed=0x31, **DESK)
    rng = O.Mt64(3)
    base = rng.pairs(5000)
    for s in range(3):
        rep = base[rng.draw(40_000) % 5000]
        g.scan_batch(rep)
        o.scan(rep)
        c = o.cells_view()
        c[1000:9000] = 0xFFFF
        g.set_cells(c[1000:9000].copy(), 1000)
        g.scan_batch(rep[:8000])
        o.scan(rep[:8000])
        assert np.array_equal(g.cells(), o.cells()), s
        g.advance_slot()
        o.advance()
        g.scan_batch(base)
        o.scan(base)
        assert np.array_equal(g.cells(), o.cells()), s


@pytest.mark.slow
def test_keyset_grows_with_the_slot_keys(gpu):
    """Slots with more keys than 0.75 x the 2^24 starting entries make the
    host grow the set at a later slot end (reallocated, starting empty), and
    small slots shrink it back; the grid stays exact across both changes.  Before the growth some probes may
    hit the bucket limit and count as fresh; after it (slot 3 on: the count
    of slot 1 is read at the end of slot 2) the count is the slot's distinct
    keys."""
    import torch

    geo = DESK
    g = _grid(gpu, geo, 0x4242, 1, k=3)
    o = O.OracleGrid(seed=0x4242, **geo)
    bucket = bucket_fn(0x4242, geo["eta"])
    rng = O.Mt64(8)
    for s in range(4):
        p = rng.pairs(18_000_000)
        p[1::5] = p[::5][: len(p[1::5])]
        before = g.fresh_pairs()
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
        o.scan(p)
        fresh, want = g.fresh_pairs() - before, distinct_keys(p, bucket)
        got, d = decode_table(g.keyset())
        assert len(np.unique(got)) == len(got), (s, "duplicate keys in the set")
        assert fresh == want if s >= 3 else fresh >= want, (s, fresh, want, len(got), int(d.max()))
        assert g.keyset().size == (1 << 24 if s < 3 else 1 << 25), s
        assert np.array_equal(g.cells(), o.cells()), s
        assert np.array_equal(g.active_counts(3), o.active_counts(3)), s
        g.advance_slot()
        o.advance()
    # small slots after the burst: the set shrinks back to 2^24 (the count of
    # slot j is read at the end of slot j + 1) and stays exact
    for s in range(4):
        p = rng.pairs(300_000)
        g.scan_batch(p)
        o.scan(p)
        assert g.keyset().size == (1 << 25 if s < 2 else 1 << 24), ("shrink", s)
        assert np.array_equal(g.cells(), o.cells()), ("shrink", s)
        g.advance_slot()
        o.advance()


M48 = (1 << 48) - 1


def perm48(x):
    """kernels.cuh cset_perm48 (numpy uint64 products wrap mod 2^64, so
    masking gives the product mod 2^48)."""
    m = np.uint64(M48)
    x = (x * np.uint64(0x9E3779B97F4B)) & m
    x ^= x >> np.uint64(23)
    x = (x * np.uint64(0xC2B2AE3D27D5)) & m
    x ^= x >> np.uint64(25)
    x = (x * np.uint64(0x165667B19E37)) & m
    x ^= x >> np.uint64(24)
    return x


def decode_table(t, bw=4):
    """Entries -> the permuted keys they name: entry = (d + 1) << rb | rem at
    bucket b, home bucket b - d (kernels.cuh scan_cset_kernel)."""
    lg = int(t.size).bit_length() - 1
    lb = bw.bit_length() - 1
    rb = 48 - (lg - lb)
    slots = np.nonzero(t)[0].astype(np.uint64)
    e = t[slots.astype(np.int64)].astype(np.uint64)
    d = (e >> np.uint64(rb)) - np.uint64(1)
    hb = ((slots >> np.uint64(lb)) - d) & np.uint64((1 << (lg - lb)) - 1)
    return (hb << np.uint64(rb)) | (e & np.uint64((1 << rb) - 1)), d


@pytest.mark.parametrize("n,dup", [(400_000, 3), (6_000_000, 5)])
def test_keyset_table_holds_each_key_once(gpu, n, dup):
    """After a slot the table holds every distinct key of it exactly once:
    decoded entries are unique and equal perm48 of the slot's keys (no key
    inserted twice by racing threads, none lost)."""
    import torch

    geo = DESK
    g = _grid(gpu, geo, 0x600d, 1, k=3)
    bucket = bucket_fn(0x600d, geo["eta"])
    rng = O.Mt64(21)
    for s in range(3):
        p = rng.pairs(n)
        p[1::dup] = p[::dup][: len(p[1::dup])]
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
        t = g.keyset()
        got, d = decode_table(t)
        keys = (p[:, 0].astype(np.uint64) << np.uint64(16)) | bucket(p[:, 1])
        want = np.unique(perm48(np.unique(keys)))
        assert len(np.unique(got)) == len(got), (s, len(got) - len(np.unique(got)))
        if len(want) <= 0.75 * t.size:  # below the growth point: no bucket-limit misses
            assert np.array_equal(np.sort(got), want), s
        else:
            assert np.isin(got, want).all(), s
        g.advance_slot()


@pytest.mark.parametrize("width", [16, 8])
@pytest.mark.parametrize("geo", [DESK, PAPER, E16], ids=["desk", "paper", "eta65536"])
def test_keyset_scan_on_narrow_grids(gpu, geo, width):
    """A narrow grid's dedup scan is the pipelined key-set kernel on its codes
    (bf16 max atomics at 16 bits, load + CAS at 8): in-window counts equal the
    oracle's over bucket-colliding traffic, and the fresh-key counter equals
    the distinct keys."""
    g = gpu.Grid(seed=0x5eed, width=width, k_max=4, **geo)
    g.scan_mode(2, -1)
    o = O.OracleGrid(seed=0x5eed, **geo)
    bucket = bucket_fn(0x5eed, geo["eta"])
    rng = O.Mt64(13)
    for s in range(4):
        p = colliding_traffic(rng, 0x5eed, geo["eta"], 2000, 3 * geo["eta"] // 2 + 1, 120_000)
        u = rng.pairs(30_000)
        before = g.fresh_pairs()
        for part in (p[:70_000], u, p[70_000:], p[:20_000]):
            g.scan_batch(part)
            o.scan(part)
        assert g.fresh_pairs() - before == distinct_keys(np.concatenate([p, u]), bucket), s
        for k in (1, 3, 4):
            assert np.array_equal(g.active_counts(k), o.active_counts(k)), (s, k)
        g.advance_slot()
        o.advance()
