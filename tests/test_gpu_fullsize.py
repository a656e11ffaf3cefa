"""Parity at BASELINE.json's full size (config C2: q16 r5 delta6 eta=65536,
an 80 GiB stamp grid on the device, 40 GiB of u16 recorders in the reference).

The compiled reference (oracle/_ref, OpenMP on all host cores) replays the
same slots: 3 slots of C2 traffic (Zipf background + injected scanners/DDoS
victims, from the repository's generator) at the full 1e8 pairs per slot:
bench.py's own trace slots 0-2 (same generator parameters).
Compared bit-exactly: per-cell R_k for several k over all 327,680
estimators, the hot sets, the reported super points and estimates, and the
full recorder contents of a random sample of 256 estimators (16.8M
recorders).  Size-independent properties are checked on the same grid:
re-scanning a slot is idempotent and the pair order does not matter.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GEO = dict(q=16, r=5, delta=6, seed=0x5eed, eta=1 << 16)
PAIRS = 100_000_000
K, THETA = 5, 1024.0


class SynthParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("hosts", C.c_uint32), ("pool", C.c_uint32),
                ("n_super", C.c_uint32), ("super_fanout", C.c_uint32),
                ("pairs_per_slot", C.c_uint64), ("shard", C.c_uint32), ("n_shards", C.c_uint32)]


def slot_pairs(L, cdf, slot):
    sp = SynthParams(0x5eed ^ 0xC2C2, 1 << 21, 16, 110, 4096, PAIRS, 0, 1)
    out = np.empty((PAIRS, 2), dtype=np.uint32)
    assert L.sspd_synth_host(C.byref(sp), cdf.ctypes.data, slot, 0, PAIRS, out.ctypes.data) == 0
    return out


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_full_size_grid_matches_reference(gpu):
    import torch

    free, _ = torch.cuda.mem_get_info(0)
    if free < 100 << 30:
        pytest.skip("needs ~95 GB of device memory")
    L = gpu.load()
    cdf = np.empty(1 << 21, dtype=np.uint64)
    assert L.sspd_synth_zipf_cdf(1 << 21, 1.1, cdf.ctypes.data) == 0
    g = gpu.Grid(**GEO)
    g.track_window(K)
    ref = O.RefGrid(GEO["q"], GEO["r"], GEO["delta"], GEO["seed"], GEO["eta"])
    workers = os.cpu_count() or 1
    rng = np.random.default_rng(5)
    for slot in range(3):
        p = slot_pairs(L, cdf, slot)
        g.scan_batch(p)
        ref.scan_alpha(p, workers)
        if slot == 1:
            # idempotence and order invariance on the full-size grid
            g.scan_batch(p[rng.permutation(len(p))[: len(p) // 2]])
        if slot < 2:
            g.advance_slot()
            ref.advance(workers)
    got_hot = g.hot_sets(K, THETA)
    ref_hot = ref.hot_sets(K, THETA)
    assert [h.tolist() for h in got_hot] == [h.tolist() for h in ref_hot]
    got = [(d.cip, d.estimate) for d in g.reconstruct_leveled(K, THETA)]
    want = [(d.cip, d.estimate) for d in ref.reconstruct(K, THETA, workers=workers)]
    assert got == want and len(got) >= 110
    # sampled estimators, bit for bit, and their R_k at several windows
    eta = GEO["eta"]
    cells_per = GEO["r"] << GEO["q"]
    sample = rng.choice(cells_per, size=256, replace=False)
    rks = {k: g.active_counts(k) for k in (1, 3, K)}
    for cell in sample:
        cell = int(cell)
        mine = g.estimator(cell >> GEO["q"], cell & ((1 << GEO["q"]) - 1))
        theirs = ref.cells_range(cell * eta, eta)
        assert np.array_equal(mine, theirs), cell
        for k, rk in rks.items():
            assert int(rk[cell]) == int((theirs < k).sum())
