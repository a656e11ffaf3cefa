"""CUDA path vs the CPU oracle, through the C ABI (include/sspd_cuda.h).

Bit-exact for the recorder grid, per-cell in-window counts, hot sets, tuple
finalisation and reported super point lists; the estimates are compared with
==, which is stricter than the 1e-6 relative tolerance BASELINE.json allows
(both sides evaluate the reference's double formula on the same integer R_k).
The cases mirror the reference's own tests (tests/test_rsea.cpp,
test_snapshot.cpp, acceptance.cpp in /root/reference/proj).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DESK = dict(q=10, r=5, delta=8, eta=256)       # desk_preset (pipeline.cpp:7-14)
PAPER = dict(q=14, r=5, delta=6, eta=2048)     # RunConfig defaults (pipeline.hpp:16-26)
ODD = dict(q=12, r=7, delta=4, eta=1000)       # non-power-of-two eta: u64 % eta path
WIDE = dict(q=16, r=8, delta=6, eta=64)        # (r-2)*delta >= 32: masked shifts
TINY = dict(q=4, r=12, delta=3, eta=40)         # 16 columns per row, non-power-of-two eta


def make_pair(gpu, geo, seed):
    g = gpu.Grid(seed=seed, **geo)
    o = O.OracleGrid(seed=seed, **geo)
    return g, o


def dets_equal(a, b):
    return [(d.cip, d.estimate) for d in a] == [(d.cip, d.estimate) for d in b]


MODES = [(0, 1), (0, 0), (1, 1), (1, 0), (2, -1), (3, -1), (-1, -1)]  # (scan mode, L1 filter)
MODE_IDS = ["bitmap+filter", "bitmap", "direct+filter", "direct", "dedup", "binned", "auto"]


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
@pytest.mark.parametrize("geo", [DESK, PAPER, ODD, WIDE, TINY],
                         ids=["desk", "paper", "odd_eta", "wide_r", "tiny_q"])
def test_scan_advance_bit_exact(gpu, geo, mode):
    g, o = make_pair(gpu, geo, 0x5eed)
    g.scan_mode(*mode)
    rng = O.Mt64(7)
    for step in range(4):
        p = rng.pairs(50_000 if geo is not PAPER else 100_000)
        g.scan_batch(p)
        o.scan(p)
        assert np.array_equal(g.cells(), o.cells()), f"grid differs after scan {step}"
        g.advance_slot()
        o.advance()
    assert np.array_equal(g.cells(), o.cells())


def test_scan_matches_compiled_reference_anchor(gpu):
    """SURVEY §8c anchor: {100k pairs; advance; 100k pairs}, mt19937_64(7),
    seed 0x5eed -> 415,545 zeros / 283,786 ones (desk) from the reference run."""
    g = gpu.Grid(seed=0x5eed, **DESK)
    rng = O.Mt64(7)
    g.scan_batch(rng.pairs(100_000)[:, ::-1])
    g.advance_slot()
    g.scan_batch(rng.pairs(100_000)[:, ::-1])
    c = g.cells()
    assert int((c == 0).sum()) == 415_545
    assert int((c == 1).sum()) == 283_786


def test_scan_batch_invariance(gpu):
    """test_rsea.cpp:78-104: batch split, permutation and empty batch."""
    rng = O.Mt64(21)
    pairs = rng.pairs(100_000)
    a = gpu.Grid(seed=0xfeed, **DESK)
    a.scan_batch(pairs)
    b = gpu.Grid(seed=0xfeed, **DESK)
    for chunk in np.array_split(pairs, 7):
        b.scan_batch(chunk)
    assert a == b
    c = gpu.Grid(seed=0xfeed, **DESK)
    c.scan_batch(pairs[np.random.default_rng(3).permutation(len(pairs))])
    assert a == c
    fresh = gpu.Grid(seed=0xfeed, **DESK)
    fresh.scan_batch(np.zeros((0, 2), np.uint32))
    assert fresh == gpu.Grid(seed=0xfeed, **DESK)
    with pytest.raises(gpu.InvalidArgument):
        fresh.scan_batch(pairs[:10], workers=0)


def test_update_touches_r_estimators(gpu):
    """test_rsea.cpp:51-76."""
    g, o = make_pair(gpu, DESK, 0xfeed)
    g.update(0xC0A80101, 0x08080808)
    o.update(0xC0A80101, 0x08080808)
    c = g.cells()
    assert np.array_equal(c, o.cells())
    assert int((c == 0).sum()) <= 5
    again = g.copy()
    again.update(0xC0A80101, 0x08080808)
    assert again == g


def test_advance_saturates(gpu):
    """test_estimator.cpp:36-47: 65534 advances -> 65534, one more -> 65535."""
    g = gpu.Grid(seed=1, **DESK)
    g.update(1, 2)
    g.advance_slot(slots=65534)
    assert int(g.cells().min()) == 65534
    g.advance_slot()
    assert int(g.cells().min()) == 65535
    assert g == gpu.Grid(seed=1, **DESK)


@pytest.mark.parametrize("k", [1, 2, 5, 30])
def test_active_counts_and_hot_sets(gpu, k):
    g, o = make_pair(gpu, DESK, 0x106)
    rng = O.Mt64(5)
    for s in range(6):
        for h in range(3):
            cip = int(rng.next()) & 0xffffffff
            pairs = np.stack([np.full(300, cip, np.uint32), rng.draw(300).astype(np.uint32)], 1)
            g.scan_batch(pairs)
            o.scan(pairs)
        p = rng.pairs(3000)
        g.scan_batch(p)
        o.scan(p)
        g.advance_slot()
        o.advance()
    assert np.array_equal(g.active_counts(k), o.active_counts(k))
    for theta in (64.0, 128.0, 300.0):
        gh, oh = g.hot_sets(k, theta), o.hot_sets(k, theta)
        assert all(np.array_equal(a, b) for a, b in zip(gh, oh))


def planted_state(gpu, geo, seed, hosts, count_lo, count_hi, noise, rng_seed):
    g, o = make_pair(gpu, geo, seed)
    rng = O.Mt64(rng_seed)
    cips = []
    for _ in range(hosts):
        cip = int(rng.next()) & 0xffffffff
        cnt = count_lo + int(rng.next()) % (count_hi - count_lo + 1)
        pairs = np.stack([np.full(cnt, cip, np.uint32), rng.draw(cnt).astype(np.uint32)], 1)
        g.scan_batch(pairs)
        o.scan(pairs)
        cips.append(cip)
    if noise:
        p = rng.pairs(noise)
        g.scan_batch(p)
        o.scan(p)
    return g, o, cips


def test_finalize_matches(gpu):
    """test_rsea.cpp:151-191, over the planted host, cold tuples and random ones."""
    g, o, cips = planted_state(gpu, DESK, 0xfeed, 3, 256, 256, 1000, 24)
    tuples = []
    for cip in cips + [0x01020304]:
        tuples.append(O.rhfg_cols(o.q, o.r, o.delta, o.seed, cip))
    rng = np.random.default_rng(0)
    hot = o.hot_sets(30, 128.0)
    for _ in range(500):
        tuples.append([int(rng.choice(h)) if len(h) else 0 for h in hot])
    t = np.array(tuples, dtype=np.uint32)
    got = g.finalize_candidates(t, 30, 128.0)
    for row, d in zip(t, got):
        ref = o.finalize(row, 30, 128.0)
        if ref is None:
            assert d is None
        else:
            assert d is not None and d.cip == ref.cip and d.estimate == ref.estimate
            assert d.r_k == ref.r_k


def test_reconstruction_equivalence(gpu):
    """acceptance.cpp:207-231 (criterion 6) against the oracle, both strategies."""
    rng = O.Mt64(106)
    for state in range(40):
        hosts = int(rng.next() % 8)
        g, o = make_pair(gpu, DESK, 0x106)
        for _ in range(hosts):
            cip = int(rng.next()) & 0xffffffff
            cnt = 32 + int(rng.next() % 512)
            pairs = np.stack([np.full(cnt, cip, np.uint32), rng.draw(cnt).astype(np.uint32)], 1)
            g.scan_batch(pairs)
            o.scan(pairs)
        p = rng.pairs(2000)
        g.scan_batch(p)
        o.scan(p)
        ref = o.reconstruct(30, 128.0)
        assert dets_equal(g.reconstruct_leveled(30, 128.0), ref), f"state {state}"
        assert dets_equal(g.reconstruct_recursive(30, 128.0), ref)


def test_reconstruct_paper_geometry(gpu):
    """20 planted supers at 2*theta over uniform background."""
    g, o = make_pair(gpu, PAPER, 0x5eed)
    rng = O.Mt64(11)
    planted = []
    for i in range(20):
        cip = int(rng.next()) & 0xffffffff
        pairs = np.stack([np.full(2048, cip, np.uint32), rng.draw(2048).astype(np.uint32)], 1)
        g.scan_batch(pairs)
        o.scan(pairs)
        planted.append(cip)
    p = rng.pairs(1_000_000)
    g.scan_batch(p)
    o.scan(p)
    ref = o.reconstruct(5, 1024.0)
    got = g.reconstruct_leveled(5, 1024.0)
    assert dets_equal(got, ref)
    assert set(planted) <= {d.cip for d in got}


def test_candidate_overflow_count(gpu):
    """test_rsea.cpp:224-238: same level and count as the reference."""
    g, o, _ = planted_state(gpu, DESK, 0xfeed, 30, 256, 256, 0, 27)
    with pytest.raises(O.CandidateOverflow) as ref:
        o.reconstruct(30, 128.0, cap=4)
    g.candidate_cap = 4
    with pytest.raises(gpu.CandidateOverflow) as got:
        g.reconstruct_leveled(30, 128.0)
    assert (got.value.level, got.value.count) == (ref.value.level, ref.value.count)
    assert str(got.value) == str(ref.value)


def test_merge_policies(gpu):
    """test_snapshot.cpp:109-144: union-min of shards == unsplit grid."""
    rng = O.Mt64(33)
    full, ofull = make_pair(gpu, DESK, 0xfeed)
    nodes = [gpu.Grid(seed=0xfeed, **DESK) for _ in range(4)]
    onodes = [O.OracleGrid(seed=0xfeed, **DESK) for _ in range(4)]
    for slot in range(3):
        p = rng.pairs(4000)
        owner = rng.draw(4000) % 4
        full.scan_batch(p)
        ofull.scan(p)
        for i in range(4):
            nodes[i].scan_batch(p[owner == i])
            onodes[i].scan(p[owner == i])
        full.advance_slot()
        ofull.advance()
        for n, on in zip(nodes, onodes):
            n.advance_slot()
            on.advance()
    m = gpu.merge_rseas(nodes, gpu.UNION_MIN)
    assert m == full
    assert np.array_equal(m.cells(), ofull.cells())
    pm = gpu.merge_rseas(nodes, gpu.PAPER_MAX)
    assert not (pm == full)
    assert np.array_equal(pm.cells(), O.OracleGrid.merge(onodes, 1).cells())
    # in place into an input
    gpu.merge_rseas(nodes, gpu.UNION_MIN, out=nodes[0])
    assert nodes[0] == full
    other = gpu.Grid(q=10, r=5, delta=8, seed=0xdef, eta=256)
    with pytest.raises(gpu.InvalidArgument, match="incompatible"):
        gpu.merge_rseas([full, other])
    with pytest.raises(gpu.InvalidArgument):
        gpu.merge_rseas([])


def test_cells_roundtrip_and_import(gpu):
    g, o = make_pair(gpu, DESK, 0x109)
    rng = O.Mt64(109)
    p = rng.pairs(20_000)
    g.scan_batch(p)
    o.scan(p)
    g.advance_slot()
    o.advance()
    c = g.cells()
    h = gpu.Grid(seed=0x109, **DESK)
    h.set_cells(c)
    assert h == g
    assert np.array_equal(h.cells(), c)
    # edits through the mutable view behave like the reference's span writes
    c2 = c.copy()
    c2[:1000] = 7
    h.set_cells(c2[:1000], 0)
    o.cells_view()[:1000] = 7
    assert np.array_equal(h.cells(), o.cells())
    assert np.array_equal(h.active_counts(8), o.active_counts(8))


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
def test_window_tracking_matches_full_count(gpu, mode):
    """The incremental in-window ring gives the same counts and reports."""
    g, o = make_pair(gpu, DESK, 0x107)
    g.scan_mode(*mode)
    g.track_window(5)
    rng = O.Mt64(8)
    for s in range(12):
        for h in range(2):
            cip = int(rng.next()) & 0xffffffff
            pairs = np.stack([np.full(200, cip, np.uint32), rng.draw(200).astype(np.uint32)], 1)
            g.scan_batch(pairs)
            o.scan(pairs)
        p = rng.pairs(4000)
        g.scan_batch(p)
        o.scan(p)
        for k in (1, 3, 5):
            assert np.array_equal(g.active_counts(k), o.active_counts(k)), (s, k)
        assert dets_equal(g.reconstruct_leveled(5, 128.0), o.reconstruct(5, 128.0))
        if s == 6:  # an import invalidates the ring; it must be rebuilt
            g.set_cells(o.cells())
        g.advance_slot()
        o.advance()


def test_invalid_config_messages(gpu):
    with pytest.raises(gpu.InvalidArgument, match="Rsea: address coverage"):
        gpu.Grid(q=8, r=5, delta=6, eta=2048)
    with pytest.raises(gpu.InvalidArgument, match="eta must be >= 2"):
        gpu.Grid(q=14, r=5, delta=6, eta=1)
    g = gpu.Grid(**DESK)
    g.update(1, 2)
    # rec::active_count does not validate k (estimator.hpp:26-31): v < 0 never
    # holds, v < k > 65535 always holds
    assert int(g.active_counts(0).max()) == 0
    assert int(g.active_counts(70000).min()) == 256


@pytest.mark.parametrize("mode", MODES, ids=MODE_IDS)
def test_repeated_pairs_and_imports_within_a_slot(gpu, mode):
    """Heavy repetition (what the dedup pair set skips) mixed with cells()
    writes and merges inside one slot: every later touch must still land."""
    g, o = make_pair(gpu, DESK, 0x77)
    g.scan_mode(*mode)
    g.track_window(4)
    rng = O.Mt64(77)
    base = rng.pairs(3000)
    for s in range(4):
        rep = base[rng.draw(20000) % 3000]  # each pair ~7 times
        g.scan_batch(rep)
        o.scan(rep)
        # reset a band of recorders to never-seen through the mutable view ...
        c = o.cells_view()
        c[: 5000] = 0xFFFF
        g.set_cells(c[:5000].copy(), 0)
        # ... and re-scan the same pairs in the same slot: they must re-touch
        g.scan_batch(rep[:5000])
        o.scan(rep[:5000])
        assert np.array_equal(g.cells(), o.cells()), s
        assert np.array_equal(g.active_counts(3), o.active_counts(3)), s
        g.advance_slot()
        o.advance()


def _hot_grid(gpu, hot_rows, geo=DESK, seed=0x31):
    """A grid whose hot columns are exactly hot_rows[row] (every bucket of
    those estimators touched this slot), built through the cells() view."""
    o = O.OracleGrid(seed=seed, **geo)
    c = o.cells_view()
    eta, ncol = geo["eta"], 1 << geo["q"]
    for row, cols in enumerate(hot_rows):
        for col in cols:
            off = (row * ncol + col) * eta
            c[off:off + eta] = 0
    g = gpu.Grid(seed=seed, **geo)
    g.set_cells(o.cells())
    return g, o


def test_candidate_buffers_grow_past_initial_allocation(gpu):
    """Level counts above the initial 2^20-tuple buffers (but under the cap)
    force the device-side re-run; results must still equal the oracle's, and
    a smaller cap must overflow at the same level with the same count."""
    rows = [range(256), range(256), range(256), range(8), range(1)]
    g, o = _hot_grid(gpu, rows)
    ref = o.reconstruct(30, 128.0)
    assert [(d.cip, d.estimate) for d in g.reconstruct_leveled(30, 128.0)] == \
        [(d.cip, d.estimate) for d in ref]
    with pytest.raises(O.CandidateOverflow) as want:
        o.reconstruct(30, 128.0, cap=5_000_000)
    g.candidate_cap = 5_000_000
    with pytest.raises(gpu.CandidateOverflow) as got:
        g.reconstruct_leveled(30, 128.0)
    assert (got.value.level, got.value.count) == (want.value.level, want.value.count)


def test_empty_hot_row_returns_nothing_even_past_cap(gpu):
    """rsea.cpp:173-174: any row without hot columns ends reconstruction
    before the level-2 cap check, however many triples rows 0-2 would give."""
    rows = [range(1024), range(1024), range(1024), range(4), []]
    g, o = _hot_grid(gpu, rows)
    g.candidate_cap = 10
    assert g.reconstruct_leveled(30, 128.0) == []
    assert o.reconstruct(30, 128.0, cap=10) == []


@pytest.mark.parametrize("mode", [(2, -1), (3, -1)], ids=["dedup", "binned"])
def test_large_device_batches(gpu, mode):
    """Device-resident batches big enough to be binned by pair-set region
    (>= 4M pairs), heavy repetition, window ring on: same grid and counts as
    the oracle."""
    import torch

    g, o = make_pair(gpu, DESK, 0x99)
    g.scan_mode(*mode)
    g.track_window(3)
    rng = O.Mt64(99)
    base = rng.pairs(200_000)
    for s in range(3):
        p = base[rng.draw(5_000_000) % 200_000]
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
        o.scan(p)
        assert np.array_equal(g.cells(), o.cells()), s
        assert np.array_equal(g.active_counts(3), o.active_counts(3)), s
        g.advance_slot()
        o.advance()


@pytest.mark.parametrize("geo", [TINY, ODD, WIDE], ids=["tiny_q", "odd_eta", "wide_r"])
def test_reconstruct_unusual_geometries(gpu, geo):
    """Hot sets and reports on geometries with few columns per row (rows
    sharing a 32-bit word of the hot bitmap), non-power-of-two eta and r=8."""
    g, o, _ = planted_state(gpu, geo, 0x5151, 4, 3 * geo["eta"], 4 * geo["eta"], 3000, 61)
    for k in (1, 5):
        theta = geo["eta"] / 2.0
        gh, oh = g.hot_sets(k, theta), o.hot_sets(k, theta)
        assert [h.tolist() for h in gh] == [h.tolist() for h in oh]
        try:
            ref = o.reconstruct(k, theta, cap=1 << 20)
        except O.CandidateOverflow as e:
            g.candidate_cap = 1 << 20
            with pytest.raises(gpu.CandidateOverflow) as got:
                g.reconstruct_leveled(k, theta)
            assert (got.value.level, got.value.count) == (e.level, e.count)
            continue
        g.candidate_cap = 1 << 20
        assert dets_equal(g.reconstruct_leveled(k, theta), ref)


EXTREMES = [dict(q=2, r=32, delta=1, eta=2),     # fewest columns, r=32, eta at its minimum
            dict(q=3, r=64, delta=1, eta=5),     # r at the reconstruct limit (64)
            dict(q=16, r=4, delta=15, eta=3),    # widest rows, delta = q - 1
            dict(q=16, r=5, delta=7, eta=1)]     # eta = 1 is invalid: checked below


@pytest.mark.parametrize("geo", EXTREMES[:3], ids=["q2_r32_eta2", "q3_r64", "q16_delta15"])
def test_extreme_geometries(gpu, geo):
    """validate_config's corners (hashing.cpp:63-87): grids, counts, hot sets
    and reports against the oracle, every slot."""
    g, o = make_pair(gpu, geo, 0xE7)
    rng = O.Mt64(0xE7)
    theta = max(1.0, geo["eta"] / 2.0)
    for s in range(5):
        p = rng.pairs(2000)
        cip = int(rng.next()) & 0xffffffff
        p = np.concatenate([p, np.stack([np.full(64, cip, np.uint32), rng.draw(64).astype(np.uint32)], 1)])
        g.scan_batch(p)
        o.scan(p)
        assert np.array_equal(g.cells(), o.cells()), s
        for k in (1, 3):
            assert np.array_equal(g.active_counts(k), o.active_counts(k)), (s, k)
            assert [h.tolist() for h in g.hot_sets(k, theta)] == [h.tolist() for h in o.hot_sets(k, theta)]
            g.candidate_cap = 1 << 16
            try:
                ref = o.reconstruct(k, theta, cap=1 << 16)
            except O.CandidateOverflow as e:
                with pytest.raises(gpu.CandidateOverflow) as got:
                    g.reconstruct_leveled(k, theta)
                assert (got.value.level, got.value.count) == (e.level, e.count)
            else:
                assert dets_equal(g.reconstruct_leveled(k, theta), ref), (s, k)
        g.advance_slot()
        o.advance()
    with pytest.raises(gpu.InvalidArgument, match="eta must be >= 2"):
        gpu.Grid(**EXTREMES[3])


def test_cabi_argument_errors(gpu):
    """Entry points reject bad arguments with the reference's exception
    classes instead of touching memory."""
    import ctypes as C

    L = gpu.load()
    g = gpu.Grid(**DESK)
    n = g.recorder_count()
    buf = np.zeros(16, dtype=np.uint16)
    ptr = buf.ctypes.data_as(C.POINTER(C.c_uint16))
    assert L.sspd_get_distances(g._h, ptr, n - 8, 16) == gpu._cabi.SSPD_OUT_OF_RANGE
    assert L.sspd_put_distances(g._h, ptr, n + 1, 1) == gpu._cabi.SSPD_OUT_OF_RANGE
    assert L.sspd_scan(g._h, None, 10, 0) == gpu._cabi.SSPD_INVALID_ARGUMENT
    assert L.sspd_scan(g._h, None, 0, 0) == gpu._cabi.SSPD_OK  # empty batch is a no-op
    with pytest.raises(gpu.InvalidArgument):
        gpu.merge_rseas([g], out=gpu.Grid(q=10, r=5, delta=8, eta=128))
    with pytest.raises(gpu.InvalidArgument):
        gpu.Grid(q=14, r=5, delta=6, eta=2048, device=99)
    # a grid on a stream of the caller's choosing still answers correctly
    import torch

    s = torch.cuda.Stream()
    g.set_stream(s.cuda_stream)
    g.update(1, 2)
    assert int((g.cells() == 0).sum()) >= 1
    g.set_stream(None)
    assert g.now == gpu.BASE_NOW


def test_fused_push_to_peer_inboxes(gpu):
    """The scan's PUSH path on one device: 'peer' inboxes are ordinary device
    buffers here (on an 8-GPU box they are NVLink-mapped symmetric memory).
    Router 1 of 3 must write exactly its new pairs, in list order, into region
    1 of the other two inboxes, nothing into its own, and leave the grid as
    the oracle's."""
    import torch

    g, o = make_pair(gpu, DESK, 0x321)
    cap = 400_000  # the new pairs plus every warp's list-block padding
    boxes = [torch.full((3 * cap, 2), -7, dtype=torch.int32, device="cuda") for _ in range(3)]
    table = torch.tensor([b.data_ptr() for b in boxes], dtype=torch.int64, device="cuda")
    g.set_exchange(2)
    g.set_push(table.data_ptr(), 3, 1, cap)
    rng = O.Mt64(321)
    base = rng.pairs(20_000)
    p = base[rng.draw(100_000) % 20_000]
    g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
    o.scan(p)
    ptr, n = g.new_pairs_ptr()
    from paper_1803_11036_b200.dist import device_view
    mine = device_view(ptr, 2 * n, g.device).view(n, 2).cpu()
    # every new pair exactly once, plus the padding of each warp's last list
    # block (kernels.cuh list_pad): copies of pairs already in the list
    distinct = np.unique(p, axis=0)
    lst = mine.numpy().view(np.uint32)
    assert len(np.unique(lst, axis=0)) == len(distinct) and n >= len(distinct)
    assert set(map(tuple, lst.tolist())) == set(map(tuple, distinct.tolist()))
    for r in (0, 2):
        got = boxes[r][cap: cap + n].cpu()
        assert torch.equal(got, mine)
        assert bool((boxes[r][:cap] == -7).all()) and bool((boxes[r][cap + n: 2 * cap] == -7).all())
    assert bool((boxes[1] == -7).all())
    assert np.array_equal(g.cells(), o.cells())
    g.set_push(0, 1, 0, 0)


def test_python_snapshot_roundtrip_matches_cli_format(gpu, tmp_path):
    """export/import in Python produce the reference file format: the same
    bytes the C++ API writes (sspd snapshot export), and a bit-exact grid."""
    import io
    import subprocess

    g, o = make_pair(gpu, DESK, 0x5eed)
    rng = O.Mt64(3)
    p = rng.pairs(30_000)
    g.scan_batch(p)
    o.scan(p)
    buf = io.BytesIO()
    gpu.export_snapshot(g, buf, k=5, theta=128, slot=0, node_id=3)
    data = buf.getvalue()
    assert len(data) == 56 + 2 * g.recorder_count()
    assert np.array_equal(np.frombuffer(data[56:], dtype="<u2"), o.cells())
    h, meta = gpu.import_snapshot(io.BytesIO(data))
    assert h == g and meta["node_id"] == 3 and meta["k"] == 5
    # the CLI (C++ API) writes the same bytes for the same scans
    trace = np.concatenate([np.zeros((len(p), 1), np.uint32), p], axis=1)
    tb = tmp_path / "t.bin"
    with open(tb, "wb") as f:
        f.write(b"SSPT" + (1).to_bytes(4, "little") + trace.astype("<u4").tobytes())
    sspd = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_1803_11036_b200", "bin", "sspd")
    out = tmp_path / "s.snap"
    subprocess.run([sspd, "snapshot", "export", str(tb), "--desk", "--k", "5", "--seed", "5eed",
                    "--node-id", "3", "-o", str(out)], check=True)
    assert out.read_bytes() == data
    with pytest.raises(RuntimeError, match="truncated payload"):
        gpu.import_snapshot(io.BytesIO(data[:-2]))


@pytest.mark.parametrize("label,shards,policy", [("single", 1, 0), ("sharded_union", 4, 0),
                                                 ("sharded_paper", 4, 1)])
def test_run_detection_matches_reference_fixture(gpu, label, shards, policy):
    """run_detection on the device against the compiled reference's reports
    on its own synth trace (tests/golden/, made by make_golden.py): same
    slots, cips and estimates, bit for bit."""
    import json

    here = os.path.dirname(os.path.abspath(__file__))
    gold = json.load(open(os.path.join(here, "golden", "golden.json")))["pipeline"]
    z = np.load(os.path.join(here, "golden", gold["trace"]))
    trace, owner = z["trace"], z["owner"]
    parts = [trace] if shards == 1 else [trace[owner == i] for i in range(shards)]
    reps = gpu.run_detection(parts, q=10, r=5, delta=8, seed=0x5eed, eta=256, k=5, theta=128.0,
                             policy=policy)
    want = gold["runs"][label]
    assert len(reps) == want["n_reports"]
    got = [[s, d.cip, d.estimate.hex()] for s, dets in reps for d in dets]
    assert got == want["rows"]
    if shards == 1:
        # the trace memory-mapped from an SSPT file: slot runs packed from the page cache
        import tempfile

        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "t.sspt")
            gpu.write_trace(trace, path)
            mapped = gpu.read_trace(path, mmap=True)
            again = gpu.run_detection([mapped], q=10, r=5, delta=8, seed=0x5eed, eta=256, k=5, theta=128.0,
                                      policy=policy)
            del mapped
        assert [[s, d.cip, d.estimate.hex()] for s, dets in again for d in dets] == want["rows"]
    if shards > 1:
        # slot runs scanned where they lie vs records selected per slot (an
        # unsorted shard takes the selection path): the same reports
        rng = np.random.default_rng(5)
        mixed = [p[rng.permutation(len(p))] for p in parts]
        again = gpu.run_detection(mixed, q=10, r=5, delta=8, seed=0x5eed, eta=256, k=5, theta=128.0,
                                  policy=policy)
        assert [[s, d.cip, d.estimate.hex()] for s, dets in again for d in dets] == want["rows"]


def test_three_routers_push_exchange_on_one_device(gpu):
    """The fused exchange end to end with the real kernels: three router grids
    on one device push their new pairs into each other's inboxes while
    scanning (parity double-buffered, as dist.PushExchange does across
    GPUs), then fold the received pairs.  Every router's grid and report must
    equal the oracle's union-min merge of the three node grids, every slot.
    (Routers run one after another: no kernel waits on another.)"""
    import torch

    world, cap = 3, 40_000
    geo = dict(DESK)
    grids = [gpu.Grid(seed=0x707, **geo) for _ in range(world)]
    nodes = [O.OracleGrid(seed=0x707, **geo) for _ in range(world)]
    inbox = [[torch.zeros((world * cap, 2), dtype=torch.int32, device="cuda") for _ in range(world)]
             for _ in range(2)]
    tables = [torch.tensor([b.data_ptr() for b in inbox[p]], dtype=torch.int64, device="cuda")
              for p in range(2)]
    for g in grids:
        g.track_window(5)
        g.set_exchange(2)
    rng = O.Mt64(707)
    base = rng.pairs(6000)
    for slot in range(4):
        par = slot & 1
        p = base[rng.draw(30_000) % 6000]
        owner = rng.draw(len(p)) % world
        counts = []
        for r, g in enumerate(grids):
            g.set_push(tables[par].data_ptr(), world, r, cap)
            mine = p[owner == r]
            g.scan_batch(torch.from_numpy(mine.view(np.int32)).cuda())
            nodes[r].scan(mine)
            counts.append(g.new_pairs_ptr()[1])
        torch.cuda.synchronize()
        for r, g in enumerate(grids):
            g.set_exchange(0)
            for src in range(world):
                if src != r and counts[src]:
                    g.scan_batch(inbox[par][r][src * cap: src * cap + counts[src]])
            g.set_exchange(2)
        want = O.OracleGrid.merge(nodes, 0)
        ref = [(d.cip, d.estimate) for d in want.reconstruct(5, 128.0)]
        for g in grids:
            assert np.array_equal(g.cells(), want.cells()), slot
            assert [(d.cip, d.estimate) for d in g.reconstruct_leveled(5, 128.0)] == ref
        for g, nd in zip(grids, nodes):
            g.advance_slot()
            nd.advance()


@pytest.mark.parametrize("mode", [(1, -1), (2, -1), (3, -1), (-1, -1)], ids=["direct", "dedup", "binned", "auto"])
def test_scan_records(gpu, mode):
    """Trace records scanned as they lie (sspd_scan_records): host arrays
    split into several staged chunks, ragged device slices, and an empty
    input -- the same grid as scanning the (cip, oip) pairs."""
    import torch

    g, o = make_pair(gpu, DESK, 0xA7)
    g.scan_mode(*mode)
    rng = O.Mt64(0xA7)
    for n in [1_200_001, 3, 0]:
        p = rng.pairs(n)
        rec = np.empty((n, 3), np.uint32)
        rec[:, 0] = np.arange(n, dtype=np.uint32)
        rec[:, 1:] = p
        g.scan_records(rec)
        o.scan(p)
    assert np.array_equal(g.cells(), o.cells())
    g.advance_slot()
    o.advance()
    p = rng.pairs(50_000)
    rec = np.concatenate([np.full((50_000, 1), 7, np.uint32), p], 1)
    dev = torch.from_numpy(rec.view(np.int32)).cuda()
    for off, n in [(1, 1), (2, 5), (9, 4321), (0, 0), (4331, 45_669)]:
        g.scan_records(dev[off:off + n])
        o.scan(p[off:off + n])
    assert np.array_equal(g.cells(), o.cells())
    assert np.array_equal(g.active_counts(2), o.active_counts(2))


@pytest.mark.parametrize("mode", [(1, -1), (2, -1), (-1, -1)], ids=["direct", "dedup", "auto"])
def test_scan_input_forms(gpu, mode):
    """Ragged and misaligned device slices (the 16-byte vector path and the
    scalar tail), pageable temporaries, and pinned host buffers the caller
    overwrites as soon as scan_batch returns (rsea.hpp:71-75 semantics)."""
    import torch

    g, o = make_pair(gpu, DESK, 0xA1)
    g.scan_mode(*mode)
    rng = O.Mt64(0xA1)
    dev = torch.from_numpy(rng.pairs(40_000).view(np.int32)).cuda()
    host = dev.cpu().numpy().view(np.uint32)
    for off, n in [(1, 1), (3, 2), (5, 3), (1, 7), (2, 1001), (7, 12_345), (0, 0)]:
        g.scan_batch(dev[off:off + n])
        o.scan(host[off:off + n])
    assert np.array_equal(g.cells(), o.cells())
    p = rng.pairs(30_000)
    g.scan_batch(p[::-1][::2])           # non-contiguous: a temporary copy, freed on return
    o.scan(np.ascontiguousarray(p[::-1][::2]))
    pinned = torch.empty((50_000, 2), dtype=torch.int32).pin_memory()
    for s in range(3):
        q = rng.pairs(50_000)
        pinned.numpy().view(np.uint32)[:] = q
        g.scan_host_ptr(pinned.data_ptr(), 50_000)
        pinned.fill_(0)                   # reused at once: the scan must already own the data
        o.scan(q)
    assert np.array_equal(g.cells(), o.cells())
    g.advance_slot()
    o.advance()
    assert np.array_equal(g.active_counts(2), o.active_counts(2))


def test_window_ring_on_fresh_imported_and_merged_grids(gpu):
    """track_window skips the stamp pass only while every stamp is 0: after
    an import, a merge or a raw stamp view it rebuilds from the stamps."""
    g, o = make_pair(gpu, DESK, 0xB2)
    rng = O.Mt64(0xB2)
    p = rng.pairs(30_000)
    o.scan(p)
    o.advance()
    o.scan(rng.pairs(10_000))
    fresh = gpu.Grid(seed=0xB2, **DESK)
    fresh.track_window(4)                      # pristine: ring zeroed, no pass
    assert int(fresh.active_counts(4).sum()) == 0
    g.set_cells(o.cells())                     # import, then track
    g.track_window(4)
    assert np.array_equal(g.active_counts(3), o.active_counts(3))
    m = gpu.merge_rseas([g, fresh])            # merge output, then track
    m.track_window(4)
    assert np.array_equal(m.active_counts(4), o.active_counts(4))
    c = gpu.Grid(seed=0xB2, **DESK)
    c.scan_batch(p)
    c.stamps_ptr()                             # raw view: the caller may rewrite stamps
    c.track_window(2)
    o2 = O.OracleGrid(seed=0xB2, **DESK)
    o2.scan(p)
    assert np.array_equal(c.active_counts(2), o2.active_counts(2))


def _shard_slot(gpu, grids, inboxes, cap, parts, k, theta):
    """One slot of the sharded union-min exchange among routers on one
    device, the collectives done in-process (dist.py ShardExchange does them
    with NCCL): scans, pushes, received scans, OR of hot bits, AND of masks."""
    import torch

    from paper_1803_11036_b200 import dist as PD

    world = len(grids)
    for g, p in zip(grids, parts):
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
    torch.cuda.synchronize()
    sent = []
    for g in grids:
        g.synchronize()
        sent.append(PD.device_view(g.shard_sent_ptr(), 2 * world, 0).view(torch.int64)[:world].tolist())
    for dst, g in enumerate(grids):
        box = inboxes[dst].view(world, cap, 2)
        for src in range(world):
            if src != dst and sent[src][dst]:
                assert sent[src][dst] <= cap
                g.shard_receive(box[src].data_ptr(), sent[src][dst])
    hot = []
    for g in grids:
        p, n = g.shard_hot(k, theta)
        hot.append(PD.device_view(p, n, 0))
    merged = hot[0].clone()
    for h in hot[1:]:
        merged |= h
    for h in hot:
        h.copy_(merged)
    torch.cuda.synchronize()
    sel = [g.shard_select(k, theta) for g in grids]
    assert len({ns for ns, _, _ in sel}) == 1
    if sel[0][0]:
        masks = [PD.device_view(p, w, 0) for _, p, w in sel]
        anded = masks[0].clone()
        for m in masks[1:]:
            anded &= m
        for m in masks:
            m.copy_(anded)
        torch.cuda.synchronize()
    return [g.shard_finish(theta) for g in grids]


@pytest.mark.parametrize("world", [1, 3, 4])
def test_sharded_routers_on_one_device(gpu, world):
    """Routers owning 1/world of the cells each: every router reports exactly
    the oracle's union-min merge, and the cells it owns equal the merged
    grid's, every slot (include/sspd_cuda.h "sharded routers")."""
    import torch

    geo = DESK
    cap = 1 << 16
    # partial grids (sspd_grid_create_sharded): each router allocates only its cells
    grids = [gpu.Grid(seed=0x5a, shard=(world, r) if world > 1 else None, **geo) for r in range(world)]
    inboxes = [torch.zeros(world * cap * 2, dtype=torch.int32, device="cuda") for _ in range(world)]
    table = torch.tensor([b.data_ptr() for b in inboxes], dtype=torch.int64, device="cuda")
    for r, g in enumerate(grids):
        g.track_window(5)
        g.set_shard(table.data_ptr(), world, r, cap)
    o = O.OracleGrid(seed=0x5a, **geo)
    rng = O.Mt64(0x5a)
    ncells = geo["r"] << geo["q"]
    for s in range(5):
        parts = []
        for r in range(world):
            p = rng.pairs(3000)
            for h in range(2 if r == 0 else 1):
                cip = 0x0A000000 + h  # super points split across routers
                p = np.concatenate([p, np.stack([np.full(90, cip, np.uint32), rng.draw(90).astype(np.uint32)], 1)])
            parts.append(p)
            o.scan(p)
        reps = _shard_slot(gpu, grids, inboxes, cap, parts, 5, 128.0)
        ref = o.reconstruct(5, 128.0)
        for rep in reps:
            assert dets_equal(rep, ref), s
        cells = o.cells()
        for r, g in enumerate(grids):
            lo = -(-r * ncells // world) * geo["eta"]
            hi = -(-(r + 1) * ncells // world) * geo["eta"]
            assert g.owned() == (lo, hi)
            assert np.array_equal(g.cells_range(lo, hi - lo), cells[lo:hi]), (s, r)
        for g in grids:
            g.advance_slot()
        o.advance()


def test_reconstruct_async_pipelines_slots(gpu):
    """sspd_reconstruct_async / _collect: the reports of slot s equal the
    oracle's for slot s although slot s+1's scan and the advance were queued
    before they were collected; collect re-reads with a larger buffer; calls
    that would clobber a queued reconstruction refuse."""
    import torch

    g, o = make_pair(gpu, DESK, 0xC3)
    g.track_window(30)
    rng = O.Mt64(0xC3)
    want = []
    got = []
    for s in range(6):
        parts = [rng.pairs(3000)]
        for h in range(1 + s % 3):
            cip = 0x0B000000 + h
            parts.append(np.stack([np.full(200, cip, np.uint32), rng.draw(200).astype(np.uint32)], 1))
        p = np.concatenate(parts)
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
        o.scan(p)
        if s:
            got.append(g.reconstruct_collect())
        g.reconstruct_async(30, 128.0)
        want.append(o.reconstruct(30, 128.0))
        if s == 2:
            with pytest.raises(gpu.InvalidArgument, match="awaits"):
                g.reconstruct_leveled(30, 128.0)
            with pytest.raises(gpu.InvalidArgument, match="awaits"):
                g.finalize_candidates(np.zeros((1, 5), np.uint32), 30, 128.0)
        g.advance_slot()
        o.advance()
    got.append(g.reconstruct_collect())
    assert len(got) == len(want)
    for s, (a, b) in enumerate(zip(got, want)):
        assert dets_equal(a, b), s
    g._report_buf = (gpu._cabi.Detection_t * 1)()  # too small: collect reads again with a larger one
    g.reconstruct_async(30, 128.0)
    assert dets_equal(g.reconstruct_collect(), o.reconstruct(30, 128.0))
    with pytest.raises(gpu.InvalidArgument, match="nothing queued"):
        g2 = gpu.Grid(seed=1, **DESK)
        g2.reconstruct_collect()


def test_counter_readbacks_leave_a_queued_reconstruction_intact(gpu):
    """bench.py's N>1 order: reconstruct_async, the next slot's scan with the
    pair list exported, new_pairs_ptr() and ==, then reconstruct_collect.  The
    counter/flag read-backs use their own pinned scratch, so the collected
    survivors (cip, R_k) are the queued slot's, equal to the oracle's."""
    import torch

    g, o = make_pair(gpu, DESK, 0xA11A)
    g.track_window(30)
    g.set_exchange(2)
    other, _ = make_pair(gpu, DESK, 0xA11A)
    rng = O.Mt64(0xA11A)
    for s in range(4):
        parts = [rng.pairs(4000)]
        for h in range(3):
            parts.append(np.stack([np.full(300, 0x0C000000 + 7 * h + s, np.uint32),
                                   rng.draw(300).astype(np.uint32)], 1))
        p = np.concatenate(parts)
        g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
        o.scan(p)
        g.reconstruct_async(30, 128.0)
        want = o.reconstruct(30, 128.0)
        assert len(want) >= 3
        nxt = rng.pairs(5000)
        g.advance_slot()
        o.advance()
        g.scan_batch(torch.from_numpy(nxt.view(np.int32)).cuda())  # export on: counts new pairs
        o.scan(nxt)
        _, n = g.new_pairs_ptr()
        assert n >= len(np.unique(nxt, axis=0))
        assert not (g == other)
        assert dets_equal(g.reconstruct_collect(), want), s
        assert np.array_equal(g.cells(), o.cells())


def test_partial_grid_refuses_whole_grid_calls(gpu):
    """A sharded router's partial grid allocates only its cells and refuses
    what needs all of them (include/sspd_cuda.h sspd_grid_create_sharded)."""
    g = gpu.Grid(seed=1, shard=(4, 1), k_max=5, **DESK)
    ncells = DESK["r"] << DESK["q"]
    lo, hi = g.owned()
    assert (lo, hi) == (-(-ncells // 4) * DESK["eta"], -(-2 * ncells // 4) * DESK["eta"])
    assert (g.cells_range(lo, hi - lo) == 0xFFFF).all()
    for call in (g.cells, lambda: g.reconstruct_leveled(5, 128.0), lambda: g.active_counts(5),
                 lambda: g.hot_sets(5, 128.0), g.copy, lambda: g.set_exchange(2),
                 lambda: g.scan_batch(np.zeros((4, 2), np.uint32)), lambda: g.cells_range(lo - 1, 2)):
        with pytest.raises(gpu.InvalidArgument):
            call()
    with pytest.raises(gpu.InvalidArgument, match="router 1 of 4"):
        g.set_shard(0, 4, 2, 16)


def _reconstruct_merged(gpu, grids, k, theta):
    """The sharded reconstruction with the collectives done in-process: OR of
    hot bits, AND of survivor masks (dist.ShardExchange.reconstruct)."""
    import torch

    from paper_1803_11036_b200 import dist as PD

    hot = []
    for g in grids:
        p, n = g.shard_hot(k, theta)
        hot.append(PD.device_view(p, n, 0))
    merged = hot[0].clone()
    for h in hot[1:]:
        merged |= h
    for h in hot:
        h.copy_(merged)
    torch.cuda.synchronize()
    sel = [g.shard_select(k, theta) for g in grids]
    assert len({ns for ns, _, _ in sel}) == 1
    if sel[0][0]:
        masks = [PD.device_view(p, w, 0) for _, p, w in sel]
        anded = masks[0].clone()
        for m in masks[1:]:
            anded &= m
        for m in masks:
            m.copy_(anded)
        torch.cuda.synchronize()
    return [g.shard_finish(theta) for g in grids]


@pytest.mark.parametrize("world", [1, 3, 4])
def test_relayed_sharded_routers_on_one_device(gpu, world):
    """Two-hop sharding: pairs go to their pair owner, which dedups the
    routers' union and relays each once to the cell owners.  Reports equal the
    oracle's union-min merge and owned cells are bit-exact, every slot."""
    import torch

    from paper_1803_11036_b200 import dist as PD

    geo = DESK
    cap = 1 << 18
    grids = [gpu.Grid(seed=0x5b, shard=(world, r) if world > 1 else None, **geo) for r in range(world)]
    in_a = [torch.zeros(world * cap * 2, dtype=torch.int32, device="cuda") for _ in range(world)]
    in_b = [torch.zeros(world * cap * 2, dtype=torch.int32, device="cuda") for _ in range(world)]
    ta = torch.tensor([b.data_ptr() for b in in_a], dtype=torch.int64, device="cuda")
    tb = torch.tensor([b.data_ptr() for b in in_b], dtype=torch.int64, device="cuda")
    for r, g in enumerate(grids):
        g.track_window(5)
        g.set_shard_relay(ta.data_ptr(), tb.data_ptr(), world, r, cap)
    o = O.OracleGrid(seed=0x5b, **geo)
    rng = O.Mt64(0x5b)
    ncells = geo["r"] << geo["q"]
    shared = rng.pairs(2000)  # pairs several routers see in the same slot
    for s in range(5):
        for r, g in enumerate(grids):
            p = np.concatenate([rng.pairs(3000), shared[r * 300: r * 300 + 1500]])
            for h in range(2 if r == 0 else 1):
                cip = 0x0A000000 + h
                p = np.concatenate([p, np.stack([np.full(90, cip, np.uint32), rng.draw(90).astype(np.uint32)], 1)])
            g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
            o.scan(p)
        torch.cuda.synchronize()
        sent = [PD.device_view(g.shard_sent_ptr(), 128, 0).view(torch.int64).tolist() for g in grids]
        for po, g in enumerate(grids):  # hop 1 -> relay (every source, the owner itself included)
            if po % 2:  # both entry points: one region at a time, and all regions in one launch
                box = in_a[po].view(world, cap, 2)
                for src in range(world):
                    if sent[src][po]:
                        assert sent[src][po] <= cap
                        g.shard_relay(box[src].data_ptr(), sent[src][po])
            else:
                g.shard_relay_regions(in_a[po].data_ptr(), cap, [sent[src][po] for src in range(world)])
        torch.cuda.synchronize()
        sent = [PD.device_view(g.shard_sent_ptr(), 128, 0).view(torch.int64).tolist() for g in grids]
        for dst, g in enumerate(grids):  # hop 2 -> cell owners
            box = in_b[dst].view(world, cap, 2)
            for src in range(world):
                if src != dst and sent[src][32 + dst]:
                    assert sent[src][32 + dst] <= cap
                    g.shard_receive(box[src].data_ptr(), sent[src][32 + dst])
        torch.cuda.synchronize()
        reps = _reconstruct_merged(gpu, grids, 5, 128.0)
        ref = o.reconstruct(5, 128.0)
        for rep in reps:
            assert dets_equal(rep, ref), s
        cells = o.cells()
        for r, g in enumerate(grids):
            lo = -(-r * ncells // world) * geo["eta"]
            hi = -(-(r + 1) * ncells // world) * geo["eta"]
            assert g.owned() == (lo, hi)
            assert np.array_equal(g.cells_range(lo, hi - lo), cells[lo:hi]), (s, r)
        for g in grids:
            g.advance_slot()
        o.advance()


def test_block_cache_reuse_and_release(gpu):
    """Closed grids leave their device blocks in the cache (sspd_release_cached);
    a new grid of the same geometry reuses them and starts pristine, as a
    freshly allocated grid does."""
    g = gpu.Grid(**DESK, seed=0x5EED)
    g.scan_batch(O.Mt64(3).pairs(50_000))
    g.close()
    h, o = make_pair(gpu, DESK, 0x5EED)  # may get g's blocks back: they must read as never seen
    assert np.array_equal(h.cells(), o.cells())
    p = O.Mt64(4).pairs(20_000)
    h.scan_batch(p)
    o.scan(p)
    assert np.array_equal(h.cells(), o.cells())
    h.close()
    assert gpu.release_cached() > 0
    assert gpu.release_cached() == 0


@pytest.mark.parametrize("world", [2, 4])
def test_relayed_routers_with_device_counts_and_peer_reduce(gpu, world):
    """dist.ShardExchange's device-driven slot, the routers on one device:
    the per-router `sent` counters gathered into one device array (the
    all-gather), relay and receive launched with the counts read by the
    kernels (sspd_shard_*_regions_dev, no host round trip), hot bits OR- and
    survivor masks AND-merged by sspd_reduce_words over the routers' copies.
    Reports equal the oracle's union-min merge, owned cells bit-exact."""
    import torch

    from paper_1803_11036_b200 import dist as PD
    from paper_1803_11036_b200.grid import reduce_words

    geo = DESK
    cap = 1 << 18
    grids = [gpu.Grid(seed=0x5c, shard=(world, r), k_max=5, **geo) for r in range(world)]
    in_a = [torch.zeros(world * cap * 2, dtype=torch.int32, device="cuda") for _ in range(world)]
    in_b = [torch.zeros(world * cap * 2, dtype=torch.int32, device="cuda") for _ in range(world)]
    ta = torch.tensor([b.data_ptr() for b in in_a], dtype=torch.int64, device="cuda")
    tb = torch.tensor([b.data_ptr() for b in in_b], dtype=torch.int64, device="cuda")
    for r, g in enumerate(grids):
        g.set_shard_relay(ta.data_ptr(), tb.data_ptr(), world, r, cap)
    o = O.OracleGrid(seed=0x5c, **geo)
    rng = O.Mt64(0x5c)
    ncells = geo["r"] << geo["q"]
    shared = rng.pairs(2000)

    def gathered(hop):  # [src * world + dst], as dist.ShardExchange._counts all-gathers it
        torch.cuda.synchronize()
        rows = [PD.device_view(g.shard_sent_ptr(), 128, 0).view(torch.int64)[32 * hop: 32 * hop + world]
                for g in grids]
        out = torch.cat(rows).contiguous()
        torch.cuda.synchronize()  # the grids' streams read it next
        return out

    for s in range(4):
        for r, g in enumerate(grids):
            p = np.concatenate([rng.pairs(3000), shared[r * 300: r * 300 + 1500]])
            cip = 0x0A000000 + (s % 2)
            p = np.concatenate([p, np.stack([np.full(150, cip, np.uint32), rng.draw(150).astype(np.uint32)], 1)])
            g.scan_batch(torch.from_numpy(p.view(np.int32)).cuda())
            o.scan(p)
        sent = gathered(0)
        for po, g in enumerate(grids):
            g.shard_relay_regions_dev(in_a[po].data_ptr(), cap, sent.data_ptr() + 8 * po, world, world)
        sent2 = gathered(1)
        for dst, g in enumerate(grids):
            g.shard_receive_regions_dev(in_b[dst].data_ptr(), cap, sent2.data_ptr() + 8 * dst, world, world, dst)
        torch.cuda.synchronize()
        assert not any(g.shard_overflow() for g in grids)
        # reconstruction: peer-reduce kernels instead of host or torch OR/AND
        hot = [g.shard_hot(5, 128.0) for g in grids]
        n = hot[0][1]
        merged = torch.empty(n, dtype=torch.int32, device="cuda")
        reduce_words(0, [p for p, _ in hot], n, "or", merged.data_ptr())
        torch.cuda.synchronize()
        for p, _ in hot:
            reduce_words(0, [merged.data_ptr()], n, "or", p)
        torch.cuda.synchronize()
        sel = [g.shard_select(5, 128.0) for g in grids]
        if sel[0][0]:
            w = sel[0][2]
            anded = torch.empty(w, dtype=torch.int32, device="cuda")
            reduce_words(0, [p for _, p, _ in sel], w, "and", anded.data_ptr())
            torch.cuda.synchronize()
            for _, p, _ in sel:
                reduce_words(0, [anded.data_ptr()], w, "and", p)
            torch.cuda.synchronize()
        ref = o.reconstruct(5, 128.0)
        assert {0x0A000000 + (s % 2)} <= {d.cip for d in ref}
        for g in grids:
            assert dets_equal(g.shard_finish(128.0), ref), s
        cells = o.cells()
        for r, g in enumerate(grids):
            lo, hi = g.owned()
            assert np.array_equal(g.cells_range(lo, hi - lo), cells[lo:hi]), (s, r)
        for g in grids:
            g.advance_slot()
        o.advance()


def test_reduce_words_matches_numpy(gpu):
    """sspd_reduce_words: OR / AND over up to 32 sources, aligned and
    misaligned, word counts not a multiple of 4."""
    import torch

    from paper_1803_11036_b200.grid import reduce_words

    rng = np.random.default_rng(3)
    for n_src, words, off in [(1, 7, 0), (3, 1000, 0), (5, 4097, 1), (32, 333, 3)]:
        host = rng.integers(0, 2**32, size=(n_src, words + 4), dtype=np.uint64).astype(np.uint32)
        dev = torch.from_numpy(host.view(np.int32)).cuda()
        srcs = [dev[i, off:].data_ptr() for i in range(n_src)]
        for op in ("or", "and"):
            out = torch.zeros(words + 1, dtype=torch.int32, device="cuda")
            reduce_words(0, srcs, words, op, out[1:].data_ptr() if off else out.data_ptr())
            torch.cuda.synchronize()
            got = (out[1:] if off else out[:words]).cpu().numpy().view(np.uint32)[:words]
            sl = host[:, off:off + words]
            want = np.bitwise_or.reduce(sl, axis=0) if op == "or" else np.bitwise_and.reduce(sl, axis=0)
            assert np.array_equal(got, want), (n_src, words, off, op)
