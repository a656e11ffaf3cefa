"""CPU model of the narrow-stamp code algebra (kernels.cuh "NARROW STAMPS",
sspd_cuda.cu sspd_advance / queue_finalize) checked against the oracle's
distances: codes rising within an epoch, the rebase before code(now) passes
`hi`, the window ring driven by old codes, and the finalize threshold.  The
GPU kernels implement the same formulas (tests/test_gpu_narrow.py checks
them on the device).
"""
import numpy as np
import pytest

from oracle import oracle as O

GEO = dict(q=4, r=12, delta=3, eta=8)  # 192 cells x 8 buckets: cheap per-slot oracle advance


class NarrowModel:
    """Recorders as codes; one 'cell' per (row, column) like the grid."""

    def __init__(self, n_cells, eta, width, K, now=65535):
        self.lo, self.hi = (0x80, 0x7F7F) if width == 16 else (1, 255)
        self.K, self.now, self.epoch0 = K, now, now
        self.codes = np.zeros((n_cells, eta), dtype=np.int64)
        self.ring = np.zeros((K, n_cells), dtype=np.int64)

    def code_now(self):
        return self.lo + (self.now - self.epoch0)

    def touch(self, cell, bucket):
        cn = self.code_now()
        old = int(self.codes[cell, bucket])
        if old >= cn:
            return
        self.codes[cell, bucket] = cn
        self.ring[self.now % self.K, cell] += 1
        if old >= self.lo and cn - old < self.K:
            self.ring[(self.now - (cn - old)) % self.K, cell] -= 1

    def advance(self):
        self.now += 1
        self.ring[self.now % self.K] = 0
        if self.code_now() > self.hi:
            cn = self.code_now()
            shift = cn - (self.lo + self.K - 1)
            live = (self.codes >= self.lo) & (cn - self.codes < self.K)
            self.codes = np.where(live, self.codes - shift, 0)
            self.epoch0 = self.now - (self.K - 1)

    def counts(self, k):
        return np.array([self.ring[(self.now - j) % self.K].copy() for j in range(k)]).sum(0)

    def counts_from_codes(self, k):
        thr = max(self.code_now() - k, self.lo - 1)
        return (self.codes > thr).sum(1)


@pytest.mark.parametrize("width,K", [(8, 1), (8, 5), (8, 30), (8, 254), (16, 64)])
def test_narrow_code_algebra_matches_distances(width, K):
    o = O.OracleGrid(seed=9, **GEO)
    n_cells = GEO["r"] << GEO["q"]
    m = NarrowModel(n_cells, GEO["eta"], width, K)
    rng = np.random.default_rng(width * 1000 + K)
    # for w=16 jump most of an epoch with idle slots (the model's advance is O(1) per slot)
    slots = 700 if width == 8 else 33000
    busy = set(range(0, slots, 1 if width == 8 else 97)) | set(range(slots - 40, slots))
    for s in range(slots):
        if s in busy:
            for _ in range(int(rng.integers(0, 40))):
                cell = int(rng.integers(0, n_cells))
                bucket = int(rng.integers(0, GEO["eta"]))
                m.touch(cell, bucket)
                o.cells_view()[cell * GEO["eta"] + bucket] = 0
            ks = {1, K, max(1, K // 2)}
            for k in ks:
                dist = o.cells_view().reshape(n_cells, GEO["eta"])
                want = (dist < k).sum(1)
                assert np.array_equal(m.counts(k), want), (s, k)
                assert np.array_equal(m.counts_from_codes(k), want), (s, k)
        m.advance()
        o.advance()
    assert m.codes.max() <= m.hi
