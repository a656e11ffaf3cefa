"""ctypes front end for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two checkers share one numpy-facing interface:

* ``OracleGrid`` -- our plain-C restatement (oracle/sspd_oracle.c,
  built to oracle/liboracle.so).
* ``RefGrid``    -- the reference itself compiled from /root/reference/proj
  (oracle/_ref/libsspd_ref.so, see oracle/Makefile), present only where it was
  built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product path
(paper_1803_11036_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsspd_ref.so")

u32p = C.POINTER(C.c_uint32)
u16p = C.POINTER(C.c_uint16)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
szp = C.POINTER(C.c_size_t)


class CandidateOverflow(RuntimeError):
    """Mirror of sspd::CandidateOverflow (rsea.hpp:38-43)."""

    def __init__(self, level: int, count: int, cap: int):
        super().__init__(
            f"candidate buffer cap exceeded at level {level}: {count} tuples, cap {cap}")
        self.level = level
        self.count = count
        self.cap = cap


@dataclass(frozen=True)
class Detection:
    cip: int
    estimate: float
    r_k: int | None = None


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class _CCfg(C.Structure):
    _fields_ = [("q", C.c_uint32), ("r", C.c_uint32), ("delta", C.c_uint32),
                ("seed", C.c_uint64)]


class _CTab(C.Structure):
    _fields_ = [("t", (C.c_uint64 * 256) * 4)]


class _CSeeds(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("h1", _CTab), ("row0", _CTab)]


class _CGrid(C.Structure):
    _fields_ = [("cfg", _CCfg), ("eta", C.c_uint32), ("seeds", _CSeeds),
                ("cells", u16p), ("n", C.c_size_t)]


class _CDet(C.Structure):
    _fields_ = [("cip", C.c_uint32), ("r_k", C.c_uint32), ("estimate", C.c_double)]


class _CRow(C.Structure):
    _fields_ = [("slot", C.c_uint64), ("det", _CDet)]


class _CMt(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        L.so_tab_hash.restype = C.c_uint64
        L.so_hash_opposite.restype = C.c_uint32
        L.so_col0.restype = C.c_uint32
        L.so_hot_cutoff.restype = C.c_size_t
        L.so_hot_cutoff.argtypes = [C.c_size_t, C.c_double]
        L.so_estimate_cardinality.restype = C.c_double
        L.so_estimate_cardinality.argtypes = [C.c_size_t, C.c_size_t]
        L.so_validate_config.argtypes = [C.POINTER(_CCfg), C.c_uint32, C.c_uint32,
                                         C.c_double, C.c_char_p, C.c_size_t]
        L.so_assemble_ip.argtypes = [u32p, C.POINTER(_CCfg), u32p]
        L.so_blocks_consistent.argtypes = [C.c_uint32, C.c_uint32, C.POINTER(_CCfg)]
        L.so_scan.argtypes = [C.POINTER(_CGrid), u32p, C.c_size_t]
        L.so_update.argtypes = [C.POINTER(_CGrid), C.c_uint32, C.c_uint32]
        L.so_hot_sets.argtypes = [C.POINTER(_CGrid), C.c_uint32, C.c_double, u32p, u32p]
        L.so_hot_sets.restype = C.c_size_t
        L.so_finalize.argtypes = [C.POINTER(_CGrid), u32p, C.c_uint32, C.c_double,
                                  C.POINTER(_CDet)]
        L.so_active_counts.argtypes = [C.POINTER(_CGrid), C.c_uint32, u32p]
        L.so_reconstruct_leveled.argtypes = [
            C.POINTER(_CGrid), C.c_uint32, C.c_double, C.c_size_t,
            C.POINTER(C.POINTER(_CDet)), szp, u32p, szp]
        L.so_reconstruct_recursive.argtypes = [
            C.POINTER(_CGrid), C.c_uint32, C.c_double, C.POINTER(C.POINTER(_CDet)), szp]
        L.so_merge.argtypes = [C.POINTER(_CGrid), C.POINTER(C.POINTER(_CGrid)),
                               C.c_size_t, C.c_int]
        L.so_run_detection.argtypes = [
            C.POINTER(_CCfg), C.c_uint32, C.c_double, C.c_uint32, C.c_uint32,
            C.c_double, C.c_int, C.c_size_t, u32p, szp, C.c_size_t, u64p,
            C.POINTER(C.POINTER(_CRow)), szp]
        L.so_free.argtypes = [C.c_void_p]
        L.so_mt64_next.restype = C.c_uint64
        L.so_mt64_seed.argtypes = [C.POINTER(_CMt), C.c_uint64]
        L.so_mt64_fill.argtypes = [C.POINTER(_CMt), u64p, C.c_size_t]
        _lib = L
    return _lib


class Mt64:
    """std::mt19937_64 replay (oracle/sspd_oracle.c so_mt64_*)."""

    def __init__(self, seed: int):
        self._s = _CMt()
        lib().so_mt64_seed(C.byref(self._s), C.c_uint64(seed))

    def next(self) -> int:
        return lib().so_mt64_next(C.byref(self._s))

    def draw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        lib().so_mt64_fill(C.byref(self._s), _ptr(out, u64p), n)
        return out

    def pairs(self, n: int) -> np.ndarray:
        """n pairs drawn as ``{(uint32)rng(), (uint32)rng()}`` (test_rsea.cpp:80-82)."""
        v = self.draw(2 * n).astype(np.uint32)
        return v.reshape(n, 2)


def cfg_struct(q, r, delta, seed=0) -> _CCfg:
    return _CCfg(q, r, delta, seed)


def h1_raw(seed: int, key: int) -> int:
    s = _CSeeds()
    lib().so_seeds_init(C.byref(s), C.c_uint64(seed))
    return lib().so_tab_hash(C.byref(s.h1), C.c_uint32(key))


def row0_raw(seed: int, key: int) -> int:
    s = _CSeeds()
    lib().so_seeds_init(C.byref(s), C.c_uint64(seed))
    return lib().so_tab_hash(C.byref(s.row0), C.c_uint32(key))


def rhfg_cols(q, r, delta, seed, cip) -> list[int]:
    """rhfg(seeds, row, cip, cfg) for every row (hashing.cpp:36-43)."""
    s = _CSeeds()
    lib().so_seeds_init(C.byref(s), C.c_uint64(seed))
    c = cfg_struct(q, r, delta, seed)
    out = []
    for row in range(r):
        v = C.c_uint32()
        lib().so_rhfg(C.byref(s), C.c_uint32(row), C.c_uint32(cip), C.byref(c), C.byref(v))
        out.append(v.value)
    return out


def hot_cutoff(eta: int, theta: float) -> int:
    return lib().so_hot_cutoff(eta, theta)


def estimate_cardinality(eta: int, r_k: int) -> float:
    return lib().so_estimate_cardinality(eta, r_k)


def validate_config(q, r, delta, eta, k, theta) -> tuple[int, str]:
    buf = C.create_string_buffer(256)
    c = cfg_struct(q, r, delta)
    n = lib().so_validate_config(C.byref(c), eta, k, theta, buf, 256)
    return n, buf.value.decode()


def assemble_ip(q, r, delta, blocks) -> int | None:
    b = np.ascontiguousarray(blocks, dtype=np.uint32)
    out = C.c_uint32()
    c = cfg_struct(q, r, delta)
    ok = lib().so_assemble_ip(_ptr(b, u32p), C.byref(c), C.byref(out))
    return out.value if ok else None


def blocks_consistent(q, r, delta, lo, hi) -> bool:
    c = cfg_struct(q, r, delta)
    return bool(lib().so_blocks_consistent(lo, hi, C.byref(c)))


class OracleGrid:
    """Rsea restated in C (u16 distance recorders, host memory)."""

    def __init__(self, q=14, r=5, delta=6, seed=0, eta=2048, _raw=None):
        self._g = _CGrid()
        if _raw is None:
            c = cfg_struct(q, r, delta, seed)
            if lib().so_grid_init(C.byref(self._g), C.byref(c), C.c_uint32(eta)) != 0:
                raise ValueError("Rsea: invalid configuration")

    def __del__(self):
        try:
            lib().so_grid_free(C.byref(self._g))
        except Exception:
            pass

    @property
    def q(self):
        return self._g.cfg.q

    @property
    def r(self):
        return self._g.cfg.r

    @property
    def delta(self):
        return self._g.cfg.delta

    @property
    def seed(self):
        return self._g.cfg.seed

    @property
    def eta(self):
        return self._g.eta

    def cells(self) -> np.ndarray:
        """Copy of the recorder array."""
        return self.cells_view().copy()

    def cells_view(self) -> np.ndarray:
        """Live view of the recorder array; valid while this grid is alive."""
        return np.ctypeslib.as_array(self._g.cells, shape=(self._g.n,))

    def copy(self) -> "OracleGrid":
        g = OracleGrid(_raw=True)
        lib().so_grid_copy(C.byref(g._g), C.byref(self._g))
        return g

    def update(self, cip: int, oip: int):
        lib().so_update(C.byref(self._g), cip, oip)

    def scan(self, pairs: np.ndarray):
        p = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        lib().so_scan(C.byref(self._g), _ptr(p, u32p), p.shape[0])

    def advance(self):
        lib().so_advance(C.byref(self._g))

    def active_counts(self, k: int) -> np.ndarray:
        out = np.empty(self.r << self.q, dtype=np.uint32)
        lib().so_active_counts(C.byref(self._g), k, _ptr(out, u32p))
        return out

    def hot_sets(self, k: int, theta: float) -> list[np.ndarray]:
        cols = np.empty(self.r << self.q, dtype=np.uint32)
        counts = np.empty(self.r, dtype=np.uint32)
        lib().so_hot_sets(C.byref(self._g), k, theta, _ptr(cols, u32p), _ptr(counts, u32p))
        out, s = [], 0
        for c in counts:
            out.append(cols[s:s + c].copy())
            s += int(c)
        return out

    def finalize(self, cols, k: int, theta: float) -> Detection | None:
        t = np.ascontiguousarray(cols, dtype=np.uint32)
        d = _CDet()
        if lib().so_finalize(C.byref(self._g), _ptr(t, u32p), k, theta, C.byref(d)):
            return Detection(d.cip, d.estimate, d.r_k)
        return None

    def _dets(self, p, n):
        res = [Detection(p[i].cip, p[i].estimate, p[i].r_k) for i in range(n)]
        lib().so_free(p)
        return res

    def reconstruct(self, k: int, theta: float, cap: int = 1 << 24,
                    leveled: bool = True) -> list[Detection]:
        p = C.POINTER(_CDet)()
        n = C.c_size_t()
        if leveled:
            lvl = C.c_uint32()
            cnt = C.c_size_t()
            rc = lib().so_reconstruct_leveled(C.byref(self._g), k, theta, cap, C.byref(p),
                                              C.byref(n), C.byref(lvl), C.byref(cnt))
            if rc == 1:
                raise CandidateOverflow(lvl.value, cnt.value, cap)
        else:
            lib().so_reconstruct_recursive(C.byref(self._g), k, theta, C.byref(p), C.byref(n))
        return self._dets(p, n.value)

    @staticmethod
    def merge(grids: list["OracleGrid"], policy: int = 0) -> "OracleGrid":
        arr = (C.POINTER(_CGrid) * len(grids))(*[C.pointer(g._g) for g in grids])
        out = OracleGrid(_raw=True)
        if lib().so_merge(C.byref(out._g), arr, len(grids), policy) != 0:
            raise ValueError(
                "merge_rseas: incompatible snapshots (seed/q/r/delta/eta differ)")
        return out

    def __eq__(self, other):
        return bool(lib().so_grid_equal(C.byref(self._g), C.byref(other._g)))


def run_detection(records: list[np.ndarray], q=14, r=5, delta=6, seed=0, eta=2048,
                  mu=1.0, k=300, start=0, theta=1024.0, policy=0, cap=1 << 24):
    """run_detection restated; records = per-shard (n,3) uint32 (ts, cip, oip).
    Returns (n_slots, list of (slot, Detection))."""
    shards = [np.ascontiguousarray(x, dtype=np.uint32).reshape(-1, 3) for x in records]
    allrec = np.concatenate(shards) if shards else np.zeros((0, 3), np.uint32)
    allrec = np.ascontiguousarray(allrec)
    off = np.zeros(len(shards) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([s.shape[0] for s in shards])
    off = off.astype(np.uintp)
    c = cfg_struct(q, r, delta, seed)
    n_slots = C.c_uint64()
    rows = C.POINTER(_CRow)()
    n = C.c_size_t()
    rc = lib().so_run_detection(C.byref(c), eta, mu, k, start, theta, policy, cap,
                                _ptr(allrec, u32p), off.ctypes.data_as(szp), len(shards),
                                C.byref(n_slots), C.byref(rows), C.byref(n))
    if rc == -1:
        raise ValueError("run_detection: invalid arguments")
    out = [(rows[i].slot, Detection(rows[i].det.cip, rows[i].det.estimate, rows[i].det.r_k))
           for i in range(n.value)]
    lib().so_free(rows)
    if rc == 1:
        raise CandidateOverflow(-1, -1, cap)
    return n_slots.value, out


# ---------------------------------------------------------------------------
# The compiled reference (oracle/_ref), when present.

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` where "
                               "/root/reference exists")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_h1_raw.restype = C.c_uint64
        L.ref_h1_raw.argtypes = [C.c_uint64, C.c_uint32]
        L.ref_row0_raw.restype = C.c_uint64
        L.ref_row0_raw.argtypes = [C.c_uint64, C.c_uint32]
        L.ref_hash_opposite.restype = C.c_uint32
        L.ref_hash_opposite.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        L.ref_hash_batch.argtypes = [C.c_uint64, u32p, C.c_size_t, u64p, u64p]
        L.ref_rhfg_cols.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, u32p,
                                    C.c_size_t, u32p]
        L.ref_assemble_ip.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, u32p]
        L.ref_blocks_consistent.argtypes = [C.c_uint32] * 5
        L.ref_hot_cutoff.restype = C.c_size_t
        L.ref_hot_cutoff.argtypes = [C.c_size_t, C.c_double]
        L.ref_estimate.restype = C.c_double
        L.ref_estimate.argtypes = [C.c_size_t, C.c_size_t]
        L.ref_validate.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                   C.c_double, C.c_char_p, C.c_size_t]
        L.ref_validate_all.restype = C.c_size_t
        L.ref_validate_all.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_double, C.c_char_p, C.c_size_t]
        L.ref_grid_create.restype = C.c_void_p
        L.ref_grid_create.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                      C.c_uint32]
        L.ref_grid_clone.restype = C.c_void_p
        L.ref_grid_clone.argtypes = [C.c_void_p]
        L.ref_grid_destroy.argtypes = [C.c_void_p]
        L.ref_grid_size.restype = C.c_size_t
        L.ref_grid_size.argtypes = [C.c_void_p]
        L.ref_update.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
        L.ref_scan.argtypes = [C.c_void_p, u32p, C.c_size_t, C.c_uint]
        L.ref_advance.argtypes = [C.c_void_p, C.c_uint]
        L.ref_scan_alpha.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint, C.c_size_t]
        L.ref_get_cells.argtypes = [C.c_void_p, u16p]
        L.ref_set_cells.argtypes = [C.c_void_p, u16p]
        L.ref_get_cells_range.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, u16p]
        L.ref_hot_sets.restype = C.c_size_t
        L.ref_hot_sets.argtypes = [C.c_void_p, C.c_uint32, C.c_double, u32p, u32p]
        L.ref_finalize.argtypes = [C.c_void_p, u32p, C.c_uint32, C.c_double, u32p, f64p]
        L.ref_reconstruct.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_double, C.c_uint,
                                      C.c_size_t, u32p, f64p, C.c_size_t, szp, u32p, szp]
        L.ref_merge.restype = C.c_void_p
        L.ref_merge.argtypes = [C.POINTER(C.c_void_p), C.c_size_t, C.c_int]
        L.ref_grid_equal.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_run_detection.argtypes = [
            C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_double,
            C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, C.c_uint, C.c_int, C.c_int,
            C.c_size_t, u32p, szp, C.c_size_t, u64p, u32p, f64p, C.c_size_t, szp, szp]
        L.ref_synth_trace.restype = C.c_size_t
        L.ref_synth_trace.argtypes = [u32p, C.c_size_t, C.c_uint32, C.c_double, C.c_uint32,
                                      C.c_uint32, C.c_uint32, C.c_uint64, C.c_double,
                                      C.c_uint32, C.c_uint32, u32p, C.c_size_t]
        _ref = L
    return _ref


class RefGrid:
    """The reference's own sspd::Rsea (compiled, namespace sspd_ref)."""

    def __init__(self, q=14, r=5, delta=6, seed=0, eta=2048, _h=None):
        if _h is None:
            _h = ref().ref_grid_create(q, r, delta, seed, eta)
            if not _h:
                raise ValueError(ref().ref_last_error().decode())
        self._h = _h
        self.q, self.r, self.delta, self.seed, self.eta = q, r, delta, seed, eta

    def __del__(self):
        try:
            ref().ref_grid_destroy(self._h)
        except Exception:
            pass

    def copy(self):
        return RefGrid(self.q, self.r, self.delta, self.seed, self.eta,
                       _h=ref().ref_grid_clone(self._h))

    def update(self, cip, oip):
        ref().ref_update(self._h, cip, oip)

    def scan(self, pairs, workers: int = 1):
        p = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        ref().ref_scan(self._h, _ptr(p, u32p), p.shape[0], workers)

    def advance(self, workers: int = 1):
        ref().ref_advance(self._h, workers)

    def scan_alpha(self, pairs: np.ndarray, workers: int, alpha: int = 1 << 15):
        """scan in the pipeline's alpha-sized batches (pipeline.cpp:58-63)."""
        p = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        ref().ref_scan_alpha(self._h, p.ctypes.data, p.shape[0], workers, alpha)

    def cells(self) -> np.ndarray:
        out = np.empty(ref().ref_grid_size(self._h), dtype=np.uint16)
        ref().ref_get_cells(self._h, _ptr(out, u16p))
        return out

    def cells_range(self, offset: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint16)
        ref().ref_get_cells_range(self._h, offset, count, _ptr(out, u16p))
        return out

    def set_cells(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.uint16)
        ref().ref_set_cells(self._h, _ptr(a, u16p))

    def hot_sets(self, k, theta):
        cols = np.empty(self.r << self.q, dtype=np.uint32)
        counts = np.empty(self.r, dtype=np.uint32)
        ref().ref_hot_sets(self._h, k, theta, _ptr(cols, u32p), _ptr(counts, u32p))
        out, s = [], 0
        for c in counts:
            out.append(cols[s:s + c].copy())
            s += int(c)
        return out

    def finalize(self, cols, k, theta):
        t = np.ascontiguousarray(cols, dtype=np.uint32)
        cip = C.c_uint32()
        est = C.c_double()
        if ref().ref_finalize(self._h, _ptr(t, u32p), k, theta, C.byref(cip), C.byref(est)):
            return Detection(cip.value, est.value)
        return None

    def reconstruct(self, k, theta, cap=1 << 24, leveled=True, workers=1):
        cap_out = 1 << 16
        cips = np.empty(cap_out, np.uint32)
        ests = np.empty(cap_out, np.float64)
        n = C.c_size_t()
        lvl = C.c_uint32()
        cnt = C.c_size_t()
        rc = ref().ref_reconstruct(self._h, int(leveled), k, theta, workers, cap,
                                   _ptr(cips, u32p), _ptr(ests, f64p), cap_out, C.byref(n),
                                   C.byref(lvl), C.byref(cnt))
        if rc == 3:
            raise CandidateOverflow(lvl.value, cnt.value, cap)
        if rc != 0:
            raise RuntimeError(ref().ref_last_error().decode())
        return [Detection(int(cips[i]), float(ests[i])) for i in range(n.value)]

    @staticmethod
    def merge(grids, policy=0):
        arr = (C.c_void_p * len(grids))(*[g._h for g in grids])
        h = ref().ref_merge(arr, len(grids), policy)
        if not h:
            raise ValueError(ref().ref_last_error().decode())
        g0 = grids[0]
        return RefGrid(g0.q, g0.r, g0.delta, g0.seed, g0.eta, _h=h)

    def __eq__(self, other):
        return bool(ref().ref_grid_equal(self._h, other._h))


def ref_validate_all(q, r, delta, eta, k, theta) -> list[str]:
    """Every message of the compiled reference's validate_config (hashing.cpp:63-87)."""
    buf = C.create_string_buffer(2048)
    n = ref().ref_validate_all(q, r, delta, eta, k, theta, buf, len(buf))
    return buf.value.decode().split("\n") if n else []


def ref_run_detection(records, q=14, r=5, delta=6, seed=0, eta=2048, mu=1.0, k=300, start=0,
                      theta=1024.0, alpha=1 << 15, workers=1, policy=0, leveled=True,
                      cap=1 << 24):
    shards = [np.ascontiguousarray(x, dtype=np.uint32).reshape(-1, 3) for x in records]
    allrec = np.ascontiguousarray(np.concatenate(shards) if shards else np.zeros((0, 3),
                                                                                 np.uint32))
    off = np.zeros(len(shards) + 1, dtype=np.uintp)
    off[1:] = np.cumsum([s.shape[0] for s in shards])
    cap_out = 1 << 20
    slots = np.empty(cap_out, np.uint64)
    cips = np.empty(cap_out, np.uint32)
    ests = np.empty(cap_out, np.float64)
    n = C.c_size_t()
    nrep = C.c_size_t()
    rc = ref().ref_run_detection(q, r, delta, seed, eta, mu, k, start, theta, alpha, workers,
                                 policy, int(leveled), cap, _ptr(allrec, u32p),
                                 off.ctypes.data_as(szp), len(shards), _ptr(slots, u64p),
                                 _ptr(cips, u32p), _ptr(ests, f64p), cap_out, C.byref(n),
                                 C.byref(nrep))
    if rc == 3:
        raise CandidateOverflow(-1, -1, cap)
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    return nrep.value, [(int(slots[i]), Detection(int(cips[i]), float(ests[i])))
                        for i in range(n.value)]


def ref_synth_trace(planted, bg_hosts, zipf, pairs_per_slot, max_distinct, slots, seed,
                    mu=1.0, k=300, start=0) -> np.ndarray:
    """The reference's synth_trace (workload.cpp:215-300) -> (n,3) uint32."""
    pl = np.ascontiguousarray(np.array(planted, dtype=np.uint32).reshape(-1, 4))
    n = ref().ref_synth_trace(_ptr(pl, u32p), pl.shape[0], bg_hosts, zipf, pairs_per_slot,
                              max_distinct, slots, seed, mu, k, start, None, 0)
    out = np.empty((n, 3), dtype=np.uint32)
    ref().ref_synth_trace(_ptr(pl, u32p), pl.shape[0], bg_hosts, zipf, pairs_per_slot,
                          max_distinct, slots, seed, mu, k, start, _ptr(out, u32p), n)
    return out


def fnv1a64(a: np.ndarray) -> int:
    """FNV-1a 64 over the little-endian bytes of an array (SURVEY §8c anchors)."""
    b = np.ascontiguousarray(a)
    L = lib()
    L.so_fnv1a64.restype = C.c_uint64
    L.so_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
    return L.so_fnv1a64(b.ctypes.data, b.nbytes)
