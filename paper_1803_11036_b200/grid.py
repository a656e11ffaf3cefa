"""Python mirror of the reference's Rsea / merge_rseas surface over the C ABI.

Method names and argument meanings follow include/sspd/rsea.hpp and
snapshot.hpp of the reference (rsea.hpp:52-114, snapshot.hpp:54), so the
parity tests read like the reference's own tests.  All work runs in the CUDA
library (lib/libsspd_cuda.so); the only host arithmetic is the reference's
double-precision hot_cutoff / estimate_cardinality formulas
(estimator.cpp:25-36), which the reports need bit-identical.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import NamedTuple

import numpy as np

from . import _cabi
from ._cabi import CandidateOverflow, check, load

BASE_NOW = 65535


class Detection(NamedTuple):
    """Detection (rsea.hpp:25-28) plus the integer in-window count behind the
    estimate.  A NamedTuple: immutable and cheap to build per report."""
    cip: int
    estimate: float
    r_k: int


# sspd_detection (include/sspd_cuda.h) as a numpy record, to read report
# buffers without one ctypes object per entry
_DET_DTYPE = np.dtype([("cip", "<u4"), ("r_k", "<u4"), ("estimate", "<f8")])


def hot_cutoff(eta: int, theta: float) -> int:
    """ceil(eta * (1 - e^(-theta/eta))) -- estimator.cpp:32-36."""
    deta = float(eta)
    return int(math.ceil(deta * (1.0 - math.exp(-theta / deta))))


def estimate_cardinality(eta: int, r_k: int) -> float:
    """-eta * ln(z0/eta), eta*ln(eta) when z0 == 0 -- estimator.cpp:25-30."""
    z0 = eta - r_k
    deta = float(eta)
    if z0 == 0:
        return deta * math.log(deta)
    return -deta * math.log(float(z0) / deta)


def device_count() -> int:
    n = C.c_int()
    check(load().sspd_device_count(C.byref(n)))
    return n.value


def device_ordinals() -> list[int]:
    """CUDA ordinals of the visible sm_100 devices (sspd_device_ordinals)."""
    out = (C.c_int * 64)()
    n = C.c_int()
    check(load().sspd_device_ordinals(out, 64, C.byref(n)))
    return list(out[:min(n.value, 64)])


def _u32(a):
    return a.ctypes.data_as(_cabi.u32p)


class Grid:
    """An RSEA grid resident on one B200 (Rsea, rsea.hpp:52-114)."""

    def __init__(self, q: int = 14, r: int = 5, delta: int = 6, seed: int = 0,
                 eta: int = 2048, device: int = 0, _handle=None, width: int = 32, k_max: int = 0,
                 shard: tuple[int, int] | None = None):
        """width 8/16 (with the window k_max): a narrow-stamp grid, exact for
        R_k with k <= k_max and the reports (sspd_grid_create_narrow).
        shard=(world, rank): a sharded router's partial grid holding only the
        cells it owns (sspd_grid_create_sharded)."""
        self._L = load()
        self.q, self.r, self.delta, self.seed, self.eta = q, r, delta, seed, eta
        if _handle is None:
            h = C.c_void_p()
            if shard is not None:
                if width != 32:
                    raise ValueError("a sharded router's grid has 32-bit stamps")
                check(self._L.sspd_grid_create_sharded(device, q, r, delta, seed, eta, k_max, shard[0],
                                                       shard[1], C.byref(h)))
            elif width == 32 and not k_max:
                check(self._L.sspd_grid_create(device, q, r, delta, seed, eta, C.byref(h)))
            else:
                check(self._L.sspd_grid_create_narrow(device, q, r, delta, seed, eta, width, k_max,
                                                      C.byref(h)))
            _handle = h
        self._h = _handle
        self.candidate_cap = 1 << 24
        self._report_buf = None

    def close(self):
        if getattr(self, "_h", None):
            self._L.sspd_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- geometry ------------------------------------------------------------
    @property
    def columns(self) -> int:
        return 1 << self.q

    def recorder_count(self) -> int:
        n = C.c_uint64()
        check(self._L.sspd_grid_info(self._h, C.byref(n), None, None))
        return n.value

    @property
    def stamp_width(self) -> tuple[int, int]:
        """(bits per stamp, tracked window k_max)."""
        w, k = C.c_uint32(), C.c_uint32()
        check(self._L.sspd_grid_stamp_width(self._h, C.byref(w), C.byref(k)))
        return w.value, k.value

    @property
    def now(self) -> int:
        v = C.c_uint32()
        check(self._L.sspd_grid_info(self._h, None, None, C.byref(v)))
        return v.value

    @property
    def device(self) -> int:
        d = C.c_int()
        check(self._L.sspd_grid_info(self._h, None, C.byref(d), None))
        return d.value

    def copy(self, device: int = -1) -> "Grid":
        h = C.c_void_p()
        check(self._L.sspd_grid_clone(self._h, device, C.byref(h)))
        g = Grid(self.q, self.r, self.delta, self.seed, self.eta, _handle=h)
        g.candidate_cap = self.candidate_cap
        return g

    # -- SCAN ------------------------------------------------------------------
    def update(self, cip: int, oip: int):
        self.scan_batch(np.array([[cip, oip]], dtype=np.uint32))

    def scan_batch(self, pairs, workers: int = 1):
        """pairs: (n,2) uint32 host array, or a CUDA tensor/array exposing
        __cuda_array_interface__ / data_ptr() on this grid's device."""
        if workers == 0:
            raise _cabi.InvalidArgument("scan_batch: workers == 0")
        if hasattr(pairs, "data_ptr") and getattr(pairs, "is_cuda", False):
            # A torch tensor: the scan runs after the work that produced it
            # on torch's current stream, and torch's later work -- including
            # the caching allocator handing this memory to a new tensor --
            # runs after the scan has read it.
            import torch

            n = pairs.numel() // 2
            cur = torch.cuda.current_stream(pairs.device)
            s = torch.cuda.ExternalStream(self.stream_handle(), device=pairs.device)
            if s.cuda_stream != cur.cuda_stream:
                s.wait_stream(cur)
            check(self._L.sspd_scan(self._h, C.c_void_p(pairs.data_ptr()), n, 1))
            if s.cuda_stream != cur.cuda_stream:
                cur.wait_stream(s)
            return
        p = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        if p.shape[0] == 0:
            return
        check(self._L.sspd_scan(self._h, p.ctypes.data_as(C.c_void_p), p.shape[0], 0))

    def scan_records(self, records):
        """(n,3) uint32 trace records (ts, cip, oip) -- a host array, or a CUDA
        tensor on this grid's device; ts is ignored (the caller picks a slot's
        records).  No host-side conversion to pairs (sspd_scan_records)."""
        if hasattr(records, "data_ptr") and getattr(records, "is_cuda", False):
            import torch

            cur = torch.cuda.current_stream(records.device)
            s = torch.cuda.ExternalStream(self.stream_handle(), device=records.device)
            if s.cuda_stream != cur.cuda_stream:
                s.wait_stream(cur)
            check(self._L.sspd_scan_records(self._h, C.c_void_p(records.data_ptr()), records.numel() // 3, 1))
            if s.cuda_stream != cur.cuda_stream:
                cur.wait_stream(s)
            return
        r = np.ascontiguousarray(records, dtype=np.uint32).reshape(-1, 3)
        if r.shape[0] == 0:
            return
        check(self._L.sspd_scan_records(self._h, r.ctypes.data_as(C.c_void_p), r.shape[0], 0))

    def scan_host_ptr(self, host_ptr: int, n_pairs: int):
        """Host (ideally pinned) buffer of n (cip, oip) pairs; copied in chunks."""
        check(self._L.sspd_scan(self._h, C.c_void_p(host_ptr), n_pairs, 0))

    def io_bytes(self, reset: bool = False) -> tuple[int, int]:
        a = C.c_uint64()
        b = C.c_uint64()
        check(self._L.sspd_grid_io_bytes(self._h, C.byref(a), C.byref(b), int(reset)))
        return a.value, b.value

    def scan_device(self, dev_ptr: int, n_pairs: int):
        check(self._L.sspd_scan(self._h, C.c_void_p(dev_ptr), n_pairs, 1))

    # -- QUIESCENT ---------------------------------------------------------
    def advance_slot(self, workers: int = 1, slots: int = 1):
        if workers == 0:
            raise _cabi.InvalidArgument("advance_slot: workers == 0")
        check(self._L.sspd_advance(self._h, slots))

    def cells(self) -> np.ndarray:
        """Host copy of all recorders as the reference's u16 distances."""
        n = self.recorder_count()
        out = np.empty(n, dtype=np.uint16)
        check(self._L.sspd_get_distances(self._h, out.ctypes.data_as(_cabi.u16p), 0, n))
        return out

    def owned(self) -> tuple[int, int]:
        """Recorders [lo, hi) this grid holds (all of them unless partial)."""
        lo, hi = C.c_uint64(), C.c_uint64()
        check(self._L.sspd_grid_owned(self._h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def cells_range(self, offset: int, count: int) -> np.ndarray:
        """Recorders [offset, offset + count) as u16 distances."""
        out = np.empty(count, dtype=np.uint16)
        check(self._L.sspd_get_distances(self._h, out.ctypes.data_as(_cabi.u16p), offset, count))
        return out

    def set_cells(self, values: np.ndarray, offset: int = 0):
        v = np.ascontiguousarray(values, dtype=np.uint16).ravel()
        check(self._L.sspd_put_distances(self._h, v.ctypes.data_as(_cabi.u16p), offset, v.size))

    def estimator(self, row: int, col: int) -> np.ndarray:
        off = ((row << self.q) + col) * self.eta
        out = np.empty(self.eta, dtype=np.uint16)
        check(self._L.sspd_get_distances(self._h, out.ctypes.data_as(_cabi.u16p), off, self.eta))
        return out

    def active_counts(self, k: int) -> np.ndarray:
        out = np.empty(self.r << self.q, dtype=np.uint32)
        check(self._L.sspd_active_counts(self._h, k, _u32(out)))
        return out

    def hot_sets(self, k: int, theta: float) -> list[np.ndarray]:
        cols = np.empty(self.r << self.q, dtype=np.uint32)
        counts = np.empty(self.r, dtype=np.uint32)
        check(self._L.sspd_hot_sets(self._h, k, hot_cutoff(self.eta, theta), _u32(cols),
                                    _u32(counts)))
        out, s = [], 0
        for c in counts:
            out.append(cols[s:s + int(c)].copy())
            s += int(c)
        return out

    def finalize_candidates(self, tuples, k: int, theta: float):
        t = np.ascontiguousarray(tuples, dtype=np.uint32).reshape(-1, self.r)
        n = t.shape[0]
        acc = np.zeros(n, dtype=np.uint8)
        cips = np.zeros(n, dtype=np.uint32)
        rks = np.zeros(n, dtype=np.uint32)
        check(self._L.sspd_finalize(self._h, _u32(t), n, k, hot_cutoff(self.eta, theta),
                                    acc.ctypes.data_as(_cabi.u8p), _u32(cips), _u32(rks)))
        return [Detection(int(cips[i]), estimate_cardinality(self.eta, int(rks[i])), int(rks[i]))
                if acc[i] else None for i in range(n)]

    def finalize_candidate(self, cols, k: int, theta: float):
        return self.finalize_candidates(np.asarray(cols).reshape(1, -1), k, theta)[0]

    def _reconstruct(self, k: int, theta: float, cap: int) -> list[Detection]:
        # the report buffer is kept across calls (reports are usually a few
        # hundred hosts at most) and regrown when a slot reports more
        while True:
            buf = self._report_buf
            if buf is None:
                buf = self._report_buf = (_cabi.Detection_t * 4096)()
            out_cap = len(buf)
            n = C.c_uint64()
            lvl = C.c_uint32()
            cnt = C.c_uint64()
            st = self._L.sspd_reconstruct(self._h, k, hot_cutoff(self.eta, theta), cap, buf,
                                          out_cap, C.byref(n), C.byref(lvl), C.byref(cnt))
            if st == _cabi.SSPD_CANDIDATE_OVERFLOW:
                raise CandidateOverflow(self._L.sspd_last_error().decode(), lvl.value, cnt.value)
            check(st)
            if n.value <= out_cap:
                rows = np.frombuffer(buf, dtype=_DET_DTYPE, count=n.value).tolist()
                return [Detection(c, e, r) for c, r, e in rows]
            self._report_buf = (_cabi.Detection_t * n.value)()

    def reconstruct_leveled(self, k: int, theta: float, workers: int = 1) -> list[Detection]:
        """Rsea::reconstruct_leveled (rsea.cpp:168-255)."""
        if workers == 0:
            raise _cabi.InvalidArgument("reconstruct_leveled: workers == 0")
        return self._reconstruct(k, theta, self.candidate_cap)

    def reconstruct_async(self, k: int, theta: float):
        """Queue reconstruct_leveled on the grid's stream and return at once
        (sspd_reconstruct_async); reconstruct_collect() returns its reports."""
        check(self._L.sspd_reconstruct_async(self._h, k, hot_cutoff(self.eta, theta), self.candidate_cap))

    def reconstruct_collect(self) -> list[Detection]:
        while True:
            buf = self._report_buf
            if buf is None:
                buf = self._report_buf = (_cabi.Detection_t * 4096)()
            n, lvl, cnt = C.c_uint64(), C.c_uint32(), C.c_uint64()
            st = self._L.sspd_reconstruct_collect(self._h, buf, len(buf), C.byref(n), C.byref(lvl),
                                                  C.byref(cnt))
            if st == _cabi.SSPD_CANDIDATE_OVERFLOW:
                raise CandidateOverflow(self._L.sspd_last_error().decode(), lvl.value, cnt.value)
            check(st)
            if n.value <= len(buf):
                rows = np.frombuffer(buf, dtype=_DET_DTYPE, count=n.value).tolist()
                return [Detection(c, e, r) for c, r, e in rows]
            self._report_buf = (_cabi.Detection_t * n.value)()  # the reports stay readable: read again

    def reconstruct_recursive(self, k: int, theta: float) -> list[Detection]:
        """Rsea::reconstruct_recursive (rsea.cpp:126-166): no candidate cap."""
        return self._reconstruct(k, theta, (1 << 64) - 1)

    def track_window(self, k_max: int):
        check(self._L.sspd_track_window(self._h, k_max))

    def stamps_ptr(self) -> tuple[int, int]:
        p = C.c_void_p()
        n = C.c_uint64()
        check(self._L.sspd_grid_stamps(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def touched_ptr(self) -> tuple[int, int]:
        p = C.c_void_p()
        n = C.c_uint64()
        check(self._L.sspd_grid_touched(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def set_exchange(self, mode: int = 1):
        """0 off, 1 touched bitmap, 2 distinct-pair list (see dist.py)."""
        check(self._L.sspd_set_exchange(self._h, int(mode)))

    def set_push(self, dev_peer_ptrs: int, world: int, rank: int, region_cap: int):
        """Fused exchange: push new pairs into peers' inboxes during the scan."""
        check(self._L.sspd_set_push(self._h, C.c_void_p(dev_peer_ptrs), world, rank, region_cap))

    def new_pairs_ptr(self) -> tuple[int, int]:
        p = C.c_void_p()
        n = C.c_uint64()
        check(self._L.sspd_grid_new_pairs(self._h, C.byref(p), C.byref(n)))
        return p.value or 0, n.value

    # -- sharded routers (include/sspd_cuda.h "sharded routers"; dist.py SHARD)
    def set_shard(self, dev_inbox_ptrs: int, world: int, rank: int, region_cap: int):
        check(self._L.sspd_set_shard(self._h, C.c_void_p(dev_inbox_ptrs), world, rank, region_cap))

    def set_shard_relay(self, dev_inbox_a: int, dev_inbox_b: int, world: int, rank: int, region_cap: int):
        check(self._L.sspd_set_shard_relay(self._h, C.c_void_p(dev_inbox_a), C.c_void_p(dev_inbox_b), world, rank,
                                           region_cap))

    def shard_relay(self, dev_ptr: int, n_pairs: int):
        check(self._L.sspd_shard_relay(self._h, C.c_void_p(dev_ptr), n_pairs))

    def shard_relay_regions(self, dev_base: int, region_stride: int, counts):
        """Relay several inbox regions (region i: counts[i] pairs at pair
        offset i * region_stride from dev_base) in one launch."""
        arr = (C.c_uint64 * len(counts))(*[int(x) for x in counts])
        check(self._L.sspd_shard_relay_regions(self._h, C.c_void_p(dev_base), region_stride, arr, len(counts)))

    def shard_relay_regions_dev(self, dev_base: int, region_stride: int, dev_counts: int, count_stride: int,
                                n_regions: int):
        """shard_relay_regions with region i's count read by the kernel from
        device memory at dev_counts[i * count_stride] (u64): no host round trip."""
        check(self._L.sspd_shard_relay_regions_dev(self._h, C.c_void_p(dev_base), region_stride,
                                                   C.c_void_p(dev_counts), count_stride, n_regions))

    def shard_receive_regions_dev(self, dev_base: int, region_stride: int, dev_counts: int, count_stride: int,
                                  n_regions: int, skip_region: int):
        """Receive n_regions inbox regions in one launch, counts in device memory."""
        check(self._L.sspd_shard_receive_regions_dev(self._h, C.c_void_p(dev_base), region_stride,
                                                     C.c_void_p(dev_counts), count_stride, n_regions, skip_region))

    def shard_overflow(self) -> bool:
        """Did a device-counted region run past its stride (since the last call)?"""
        f = C.c_int()
        check(self._L.sspd_shard_overflow(self._h, C.byref(f)))
        return bool(f.value)

    def shard_sent_ptr(self) -> int:
        """Device u64[world]: pairs this router pushed to each owner this slot."""
        p = C.c_void_p()
        check(self._L.sspd_shard_sent(self._h, C.byref(p)))
        return p.value

    def shard_receive(self, dev_ptr: int, n_pairs: int):
        check(self._L.sspd_shard_receive(self._h, C.c_void_p(dev_ptr), n_pairs))

    def shard_hot(self, k: int, theta: float) -> tuple[int, int]:
        """(device pointer, u32 words) of this router's hot bits, to OR-merge."""
        p, n = C.c_void_p(), C.c_uint64()
        check(self._L.sspd_shard_hot(self._h, k, hot_cutoff(self.eta, theta), C.byref(p), C.byref(n)))
        return p.value, n.value

    def shard_select(self, k: int, theta: float, cap: int | None = None) -> tuple[int, int, int]:
        """(survivors, device pointer, u32 words) of the per-survivor bucket
        masks, to AND-merge; raises CandidateOverflow like reconstruct."""
        ns, p, w = C.c_uint64(), C.c_void_p(), C.c_uint64()
        lvl, cnt = C.c_uint32(), C.c_uint64()
        cap = self.candidate_cap if cap is None else cap
        st = self._L.sspd_shard_select(self._h, k, hot_cutoff(self.eta, theta), cap, C.byref(ns), C.byref(p),
                                       C.byref(w), C.byref(lvl), C.byref(cnt))
        if st == _cabi.SSPD_CANDIDATE_OVERFLOW:
            raise CandidateOverflow(self._L.sspd_last_error().decode(), lvl.value, cnt.value)
        check(st)
        return ns.value, p.value or 0, w.value

    def shard_finish(self, theta: float) -> list[Detection]:
        while True:
            buf = self._report_buf
            if buf is None:
                buf = self._report_buf = (_cabi.Detection_t * 4096)()
            n = C.c_uint64()
            check(self._L.sspd_shard_finish(self._h, hot_cutoff(self.eta, theta), buf, len(buf), C.byref(n)))
            if n.value <= len(buf):
                rows = np.frombuffer(buf, dtype=_DET_DTYPE, count=n.value).tolist()
                return [Detection(c, e, r) for c, r, e in rows]
            self._report_buf = (_cabi.Detection_t * n.value)()

    def fresh_pairs(self) -> int:
        """Keys the pipelined dedup scan found new to their slot, since creation:
        (cip, bucket) keys on the key-set scan (eta <= 2^16), else (cip, oip) pairs."""
        n = C.c_uint64()
        check(self._L.sspd_grid_fresh_pairs(self._h, C.byref(n)))
        return n.value

    def keyset(self) -> np.ndarray | None:
        """The per-slot key set's entries (a host copy; None before the first
        key-set scan)."""
        p, lg = C.c_void_p(), C.c_uint32()
        check(self._L.sspd_grid_keyset(self._h, C.byref(p), C.byref(lg)))
        if not p.value:
            return None
        from .dist import device_view
        return device_view(p.value, 1 << lg.value, self.device).cpu().numpy().view(np.uint32)

    def scan_mode(self, mode: int = -1, filter: int = -1):
        """Scan strategy (include/sspd_cuda.h sspd_scan_mode): 0 = deferred bitmap,
        1 = direct stamping, 2 = direct behind the per-slot pair set, 3 = 2 after
        binning large device batches, -1 = auto; filter 0/1 = L1 duplicate probe
        (-1 keeps).  Narrow-stamp grids run 0 as 1 and 3 as 2."""
        check(self._L.sspd_scan_mode(self._h, mode, filter))

    def commit(self):
        check(self._L.sspd_commit(self._h))

    def synchronize(self):
        check(self._L.sspd_grid_synchronize(self._h))

    def stream_handle(self) -> int:
        """The cudaStream_t (as an int) the grid queues its work on."""
        p = C.c_void_p()
        check(self._L.sspd_grid_stream(self._h, C.byref(p)))
        return p.value or 0

    def set_stream(self, stream_ptr: int | None):
        check(self._L.sspd_grid_set_stream(self._h, C.c_void_p(stream_ptr or 0)))

    # profiling -----------------------------------------------------------
    def profile(self, on: bool = True):
        check(self._L.sspd_profile_enable(self._h, int(on)))

    def profile_reset(self):
        check(self._L.sspd_profile_reset(self._h))

    def profile_read(self, kernel: str | None = None) -> tuple[float, int, int]:
        ms = C.c_double()
        n = C.c_uint64()
        u = C.c_uint64()
        check(self._L.sspd_profile_read(self._h, kernel.encode() if kernel else None,
                                        C.byref(ms), C.byref(n), C.byref(u)))
        return ms.value, n.value, u.value

    def __eq__(self, other: "Grid") -> bool:
        e = C.c_int()
        check(self._L.sspd_equal(self._h, other._h, C.byref(e)))
        return bool(e.value)


def merge_rseas(grids: list[Grid], policy: int = _cabi.UNION_MIN, out: Grid | None = None,
                device: int | None = None) -> Grid:
    """merge_rseas (snapshot.hpp:54): a new grid (or `out`) holding the
    element-wise union-min / paper-max of the inputs."""
    if not grids:
        raise _cabi.InvalidArgument("merge_rseas: empty set")
    g0 = grids[0]
    if out is None:
        out = Grid(g0.q, g0.r, g0.delta, g0.seed, g0.eta,
                   device=g0.device if device is None else device)
        out.candidate_cap = g0.candidate_cap
    arr = (C.c_void_p * len(grids))(*[g._h for g in grids])
    check(load().sspd_merge(arr, len(grids), policy, out._h))
    return out


SNAPSHOT_MAGIC = b"RSEA"
SNAPSHOT_VERSION = 1
SNAPSHOT_HEADER = 56


def export_snapshot(grid: Grid, f, k: int = 0, theta: int = 0, slot: int = 0, node_id: int = 0,
                    chunk: int = 1 << 22):
    """export_snapshot (snapshot.hpp:30-41; snapshot.cpp:36-68): 56-byte
    little-endian header, then every recorder as a u16 distance in (row,
    column, bucket) order, streamed from the device in chunks."""
    import struct

    f.write(SNAPSHOT_MAGIC + struct.pack("<IQIIIIIIQI4x", SNAPSHOT_VERSION, grid.seed, grid.q,
                                         grid.r, grid.delta, grid.eta, k, theta, slot, node_id))
    n = grid.recorder_count()
    buf = np.empty(min(chunk, n), dtype=np.uint16)
    for pos in range(0, n, chunk):
        cnt = min(chunk, n - pos)
        check(load().sspd_get_distances(grid._h, buf.ctypes.data_as(_cabi.u16p), pos, cnt))
        f.write(buf[:cnt].astype("<u2").tobytes())


def import_snapshot(f, device: int = 0, chunk: int = 1 << 22):
    """import_snapshot (snapshot.cpp:70-115): returns (grid, meta dict) with
    the reference's validation messages."""
    import struct

    h = f.read(SNAPSHOT_HEADER)
    if len(h) != SNAPSHOT_HEADER:
        raise RuntimeError("import_snapshot: truncated header")
    if h[:4] != SNAPSHOT_MAGIC:
        raise RuntimeError("import_snapshot: bad magic")
    (version, seed, q, r, delta, eta, k, theta, slot, node_id) = struct.unpack("<IQIIIIIIQI4x", h[4:])
    if version != SNAPSHOT_VERSION:
        raise RuntimeError(f"import_snapshot: unsupported version {version}")
    g = Grid(q, r, delta, seed, eta, device=device)
    n = g.recorder_count()
    for pos in range(0, n, chunk):
        cnt = min(chunk, n - pos)
        raw = f.read(2 * cnt)
        if len(raw) != 2 * cnt:
            raise RuntimeError(f"import_snapshot: truncated payload, expected {2 * n} bytes, "
                               f"got {2 * pos + len(raw)}")
        g.set_cells(np.frombuffer(raw, dtype="<u2"), pos)
    meta = dict(seed=seed, q=q, r=r, delta=delta, eta=eta, k=k, theta=theta, slot=slot,
                node_id=node_id)
    return g, meta


def exact_counts(segments, min_count: int = 1, distinct_hint: int = 0, device: int = 0,
                 stream_ptr: int | None = None) -> dict:
    """Exact distinct-oip counts per cip over the union of device segments of
    (cip, oip) pairs (torch CUDA tensors shaped (n, 2)), like exact_counts
    for one window (workload.cpp:180-213).  Returns {cip: count >= min_count}."""
    segs = [s for s in segments if s.numel()]
    ptrs = (C.c_void_p * max(len(segs), 1))(*[s.data_ptr() for s in segs])
    sizes = (C.c_uint64 * max(len(segs), 1))(*[s.numel() // 2 for s in segs])
    cap = 1 << 16
    while True:
        cips = np.empty(cap, dtype=np.uint32)
        counts = np.empty(cap, dtype=np.uint32)
        n = C.c_uint64()
        check(load().sspd_exact_counts(device, ptrs, sizes, len(segs), distinct_hint, min_count,
                                       _u32(cips), _u32(counts), cap, C.byref(n),
                                       C.c_void_p(stream_ptr or 0)))
        if n.value <= cap:
            return {int(c): int(k) for c, k in zip(cips[:n.value], counts[:n.value])}
        cap = int(n.value)


def reduce_words(device: int, srcs: list[int], words: int, op: str, dst: int, stream: int = 0):
    """dst = OR ("or") / AND ("and") of the u32 arrays at the device pointers
    srcs (peers' buffers allowed), one kernel (sspd_reduce_words)."""
    arr = (C.c_void_p * len(srcs))(*[C.c_void_p(int(p)) for p in srcs])
    check(load().sspd_reduce_words(device, arr, len(srcs), words, {"or": 0, "and": 1}[op], C.c_void_p(dst),
                                   C.c_void_p(stream)))


def checked_status(device: int = 0, reset: bool = True) -> tuple[int, int]:
    """(first failing kernels.cuh line, failures) of the checked build's device
    bounds/invariant checks; raises InvalidArgument on the product build."""
    line, n = C.c_uint32(), C.c_uint64()
    check(load().sspd_checked_status(device, C.byref(line), C.byref(n), 1 if reset else 0))
    return line.value, n.value


def launch_count() -> int:
    return int(load().sspd_launch_count())


def release_cached(device: int = -1) -> int:
    """Free the device blocks closed grids left for reuse (sspd_release_cached);
    returns the bytes freed.  Call before handing the memory to torch."""
    n = C.c_uint64()
    check(load().sspd_release_cached(device, C.byref(n)))
    return n.value
