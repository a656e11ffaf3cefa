"""Narrow-stamp grids (8/16-bit stamps, BASELINE config C4's stamp-width axis)
against the CPU oracle.

A narrow grid is exact for the in-window counts R_k with k <= k_max and for
everything derived from them (hot sets, finalize, reconstruction reports);
these tests check that, bit for bit, across many code epochs and the rebase
passes between them (kernels.cuh "NARROW STAMPS"), in every scan mode and
geometry class.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DESK = dict(q=10, r=5, delta=8, eta=256)       # desk_preset (pipeline.cpp:7-14)
ODD = dict(q=12, r=7, delta=4, eta=1000)       # non-power-of-two eta
TINY = dict(q=4, r=12, delta=3, eta=40)        # 16 columns per row


def dets_equal(a, b):
    return [(d.cip, d.estimate) for d in a] == [(d.cip, d.estimate) for d in b]


def recon_equal(gpu, g, o, k, theta):
    """Same reports, or the same CandidateOverflow (level and count)."""
    try:
        ref = o.reconstruct(k, theta)
    except O.CandidateOverflow as e:
        with pytest.raises(gpu.CandidateOverflow) as got:
            g.reconstruct_leveled(k, theta)
        return (got.value.level, got.value.count) == (e.level, e.count)
    return dets_equal(g.reconstruct_leveled(k, theta), ref)


def oracle_advance(o, n):
    """n advance_slot calls on the oracle (saturating distances)."""
    if n <= 4:
        for _ in range(n):
            o.advance()
        return
    v = o.cells_view()
    v[:] = np.minimum(v.astype(np.uint32) + n, 0xFFFF).astype(np.uint16)


def slot_traffic(rng, hosts, fanout, noise):
    parts = []
    for _ in range(hosts):
        cip = int(rng.next()) & 0xffffffff
        parts.append(np.stack([np.full(fanout, cip, np.uint32), rng.draw(fanout).astype(np.uint32)], 1))
    parts.append(rng.pairs(noise))
    return np.concatenate(parts)


@pytest.mark.parametrize("mode", [1, 2, "pairset", -1], ids=["direct", "dedup", "dedup_pairset", "auto"])
@pytest.mark.parametrize("geo", [DESK, ODD, TINY], ids=["desk", "odd_eta", "tiny_q"])
def test_width8_counts_and_reports_across_wraps(gpu, geo, mode, monkeypatch):
    """600 slots at w=8: epochs of 255 then 226 slots (K = 30), so two rebase
    passes; a recurring host that keeps cells hot, then goes quiet.  dedup:
    the key-set scan on byte codes; dedup_pairset: the narrow pair-set scan."""
    k_max = 30
    if mode == "pairset":
        monkeypatch.setenv("SSPD_CSET", "0")
        mode = 2
    g = gpu.Grid(seed=0x5eed, width=8, k_max=k_max, **geo)
    g.scan_mode(mode, -1)
    o = O.OracleGrid(seed=0x5eed, **geo)
    rng = O.Mt64(0x8b17)
    fixed = int(rng.next()) & 0xffffffff
    theta = 128.0 if geo["eta"] >= 256 else 16.0
    for s in range(600):
        p = slot_traffic(rng, 1 if s % 3 == 0 else 0, 150 if geo["eta"] >= 256 else 12,
                         400 if geo["eta"] >= 256 else 8)
        if s % 50 < 20:  # a host that is a super point for a while, then goes quiet
            fan = 60 if geo["eta"] >= 256 else 6
            p = np.concatenate([p, np.stack([np.full(fan, fixed, np.uint32),
                                             rng.draw(fan).astype(np.uint32)], 1)])
        g.scan_batch(p)
        o.scan(p)
        if s % 37 == 0 or s in (253, 254, 255, 256, 479, 480, 481, 482, 599):
            for k in (1, 7, k_max):
                assert np.array_equal(g.active_counts(k), o.active_counts(k)), (s, k)
            assert recon_equal(gpu, g, o, k_max, theta), s
            assert recon_equal(gpu, g, o, 5, theta), s
        g.advance_slot()
        o.advance()


@pytest.mark.parametrize("mode", [1, 2, "pairset"], ids=["direct", "dedup", "dedup_pairset"])
def test_width16_counts_across_a_wrap(gpu, mode, monkeypatch):
    """w=16 (bf16-ordered codes, epochs of ~32K slots): bulk advances carry
    the grid across several rebases while recorders of every age are kept.
    dedup: the pipelined key-set scan on bf16 codes; dedup_pairset: the
    narrow scan behind the 8-byte pair set ($SSPD_CSET=0)."""
    k_max = 64
    if mode == "pairset":
        monkeypatch.setenv("SSPD_CSET", "0")
        mode = 2
    g = gpu.Grid(seed=0x77, width=16, k_max=k_max, **DESK)
    g.scan_mode(mode, -1)
    o = O.OracleGrid(seed=0x77, **DESK)
    rng = O.Mt64(16)
    gaps = [1, 1, 3, 40, 30000, 2, 2400, 1, 63, 64, 65, 32380, 7, 1, 32447, 1]
    for i, gap in enumerate(gaps):
        p = slot_traffic(rng, 2, 200, 3000)
        g.scan_batch(p)
        o.scan(p)
        for k in (1, 2, 30, k_max):
            assert np.array_equal(g.active_counts(k), o.active_counts(k)), (i, k)
        assert dets_equal(g.reconstruct_leveled(k_max, 128.0), o.reconstruct(k_max, 128.0)), i
        g.advance_slot(slots=gap)
        oracle_advance(o, gap)
    assert g.now - 65535 == sum(gaps)


@pytest.mark.parametrize("width", [8, 16])
def test_narrow_finalize_and_hot_sets(gpu, width):
    g = gpu.Grid(seed=0xfeed, width=width, k_max=30, **DESK)
    o = O.OracleGrid(seed=0xfeed, **DESK)
    rng = O.Mt64(24)
    cips = []
    for s in range(5):
        p = slot_traffic(rng, 3, 256, 1000)
        cips += [int(c) for c in np.unique(p[:-1000, 0])]
        g.scan_batch(p)
        o.scan(p)
        g.advance_slot()
        o.advance()
    for k in (1, 5, 30):
        for theta in (64.0, 128.0, 300.0):
            assert all(np.array_equal(a, b) for a, b in zip(g.hot_sets(k, theta), o.hot_sets(k, theta)))
    tuples = [O.rhfg_cols(o.q, o.r, o.delta, o.seed, c) for c in cips + [0x01020304]]
    npr = np.random.default_rng(0)
    hot = o.hot_sets(30, 128.0)
    tuples += [[int(npr.choice(h)) if len(h) else 0 for h in hot] for _ in range(300)]
    t = np.array(tuples, dtype=np.uint32)
    for row, d in zip(t, g.finalize_candidates(t, 30, 128.0)):
        ref = o.finalize(row, 30, 128.0)
        assert (d is None) == (ref is None)
        if ref is not None:
            assert (d.cip, d.estimate, d.r_k) == (ref.cip, ref.estimate, ref.r_k)


def test_narrow_grid_equals_wide_grid_reports(gpu):
    """The three widths give the same counts and reports on the same traffic."""
    grids = [gpu.Grid(seed=3, width=w, k_max=16, **DESK) for w in (8, 16, 32)]
    rng = O.Mt64(99)
    for s in range(300):
        p = slot_traffic(rng, 1 if s % 4 == 0 else 0, 180, 500)
        for g in grids:
            g.scan_batch(p)
        if s % 29 == 0:
            ref = grids[2].active_counts(16)
            rep = grids[2].reconstruct_leveled(16, 128.0)
            for g in grids[:2]:
                assert np.array_equal(g.active_counts(16), ref)
                assert dets_equal(g.reconstruct_leveled(16, 128.0), rep)
        for g in grids:
            g.advance_slot()
    assert [g.stamp_width for g in grids] == [(8, 16), (16, 16), (32, 16)]


def test_narrow_grid_refuses_what_it_cannot_answer(gpu):
    g = gpu.Grid(seed=1, width=8, k_max=10, **DESK)
    g.scan_batch(O.Mt64(1).pairs(1000))
    with pytest.raises(gpu.InvalidArgument, match="8-bit stamps"):
        g.cells()
    with pytest.raises(gpu.InvalidArgument, match="exceeds the window"):
        g.active_counts(11)
    with pytest.raises(gpu.InvalidArgument, match="8-bit stamps"):
        gpu.merge_rseas([g, g])
    with pytest.raises(gpu.InvalidArgument, match="8-bit stamps"):
        g.track_window(20)
    g.track_window(10)  # its own window: a no-op
    assert g.active_counts(0).sum() == 0
    assert int(g.active_counts(1 << 20).min()) == 256  # k > 65535: every bucket
    with pytest.raises(gpu.InvalidArgument, match="needs more than 8-bit"):
        gpu.Grid(seed=1, width=8, k_max=255, **DESK)
    with pytest.raises(gpu.InvalidArgument, match="needs more than 16-bit"):
        gpu.Grid(seed=1, width=16, k_max=32512, **DESK)
    with pytest.raises(gpu.InvalidArgument, match="stamp width"):
        gpu.Grid(seed=1, width=12, k_max=10, **DESK)
