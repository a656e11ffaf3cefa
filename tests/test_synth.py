"""The workload generator (csrc/synth.h) is bit-identical across its three
builds: host code in the CUDA library, the host-only library used by the
reference arm, and the device kernel (GPU test)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1803_11036_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SYNTH = os.path.join(ROOT, "oracle", "libsynth_host.so")


class Params(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("hosts", C.c_uint32), ("pool", C.c_uint32),
                ("n_super", C.c_uint32), ("super_fanout", C.c_uint32),
                ("pairs_per_slot", C.c_uint64), ("shard", C.c_uint32), ("n_shards", C.c_uint32)]


def cases():
    yield Params(0x5eed, 1 << 16, 16, 11, 512, 200_000, 0, 1)      # Zipf + injected
    yield Params(0xabc, 1, 0, 20, 2048, 100_000, 0, 1)              # uniform (C1)
    yield Params(0x5eed, 1 << 16, 16, 11, 512, 400_000, 2, 4)       # router shard 2 of 4


def host_pairs(lib_fn_cdf, lib_fn_pairs, p, slot, n):
    cdf = np.empty(p.hosts, dtype=np.uint64)
    assert lib_fn_cdf(C.c_uint32(p.hosts), C.c_double(1.1), C.c_void_p(cdf.ctypes.data)) == 0
    out = np.empty((n, 2), dtype=np.uint32)
    assert lib_fn_pairs(C.byref(p), C.c_void_p(cdf.ctypes.data), C.c_uint64(slot), C.c_uint64(0),
                        C.c_uint64(n), C.c_void_p(out.ctypes.data)) == 0
    return cdf, out


def test_host_builds_agree_and_shard_partition():
    L = P.load()
    S = C.CDLL(SYNTH)
    for p in cases():
        n = p.pairs_per_slot // p.n_shards
        cdf_a, a = host_pairs(L.sspd_synth_zipf_cdf, L.sspd_synth_host, p, 3, n)
        cdf_b, b = host_pairs(S.sspd_synth_zipf_cdf_host, S.sspd_synth_pairs_host, p, 3, n)
        assert np.array_equal(cdf_a, cdf_b)
        assert np.array_equal(a, b)
        assert cdf_a[-1] == 1 << 63 and np.all(np.diff(cdf_a.astype(np.float64)) >= 0)
    # the injected super points carry exactly super_fanout distinct opposites
    p = next(cases())
    _, a = host_pairs(L.sspd_synth_zipf_cdf, L.sspd_synth_host, p, 0, p.pairs_per_slot)
    inj = a[: p.n_super * p.super_fanout]
    for i in range(p.n_super):
        cip = L.sspd_synth_super_cip(C.byref(p), i)
        rows = inj[inj[:, 0] == cip]
        assert len(np.unique(rows[:, 1])) == p.super_fanout
    # background hosts never exceed their pool
    bg = a[p.n_super * p.super_fanout:]
    keys = np.unique(bg, axis=0)
    _, per_host = np.unique(keys[:, 0], return_counts=True)
    assert per_host.max() <= p.pool


@pytest.mark.gpu
def test_device_generator_matches_host(gpu):
    import torch

    L = P.load()
    for p in cases():
        n = p.pairs_per_slot // p.n_shards
        cdf, want = host_pairs(L.sspd_synth_zipf_cdf, L.sspd_synth_host, p, 7, n)
        dcdf = torch.from_numpy(cdf.view(np.int64)).cuda()
        out = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        P._cabi.check(L.sspd_synth_device(0, C.byref(p), C.c_void_p(dcdf.data_ptr()), 7, 0, n,
                                          C.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want)


@pytest.mark.gpu
def test_exact_counts_on_device_match_host(gpu):
    """sspd_exact_counts == the union-of-sets definition (workload.cpp:180-213)
    over several overlapping segments, including cip 0xFFFFFFFF and the pair
    equal to the empty-key marker."""
    import torch

    rng = np.random.default_rng(17)
    segs = []
    for n in (50_000, 80_000, 3):
        cip = rng.integers(0, 3000, n).astype(np.uint32)
        oip = rng.integers(0, 400, n).astype(np.uint32)
        segs.append(np.stack([cip, oip], 1))
    segs[2][:] = [[0xFFFFFFFF, 0xFFFFFFFF], [0xFFFFFFFF, 7], [5, 0xFFFFFFFF]]
    allp = np.concatenate(segs)
    uniq = np.unique(allp, axis=0)
    cips, cnt = np.unique(uniq[:, 0], return_counts=True)
    want = {int(c): int(k) for c, k in zip(cips, cnt)}
    dev = [torch.from_numpy(s.view(np.int32)).cuda() for s in segs]
    assert gpu.exact_counts(dev) == want
    assert gpu.exact_counts(dev, min_count=200) == {c: k for c, k in want.items() if k >= 200}
    with pytest.raises(gpu.OutOfRange):
        gpu.exact_counts(dev, distinct_hint=16)   # table too small: an error, never a wrong count
