"""ctypes declarations for the C ABI in include/sspd_cuda.h.

The library is built in-tree (paper_1803_11036_b200/lib/libsspd_cuda.so, see
csrc/Makefile and __graft_entry__.build()).  There is no CPU fallback: if the
library is missing or no sm_100 device is visible, every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSPD_LIB") or os.path.join(HERE, "lib", "libsspd_cuda.so")

SSPD_OK = 0
SSPD_INVALID_ARGUMENT = 1
SSPD_OUT_OF_RANGE = 2
SSPD_CANDIDATE_OVERFLOW = 3
SSPD_CUDA_ERROR = 4
SSPD_NO_DEVICE = 5

UNION_MIN = 0
PAPER_MAX = 1

u32p = C.POINTER(C.c_uint32)
u16p = C.POINTER(C.c_uint16)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)
grid_p = C.c_void_p


class Detection_t(C.Structure):
    _fields_ = [("cip", C.c_uint32), ("r_k", C.c_uint32), ("estimate", C.c_double)]


# name -> (restype, argtypes); also the list of symbols include/sspd_cuda.h
# declares (tests/test_cabi_symbols.py checks the .so exports every one).
SIGNATURES = {
    "sspd_abi_version": (C.c_int, []),
    "sspd_last_error": (C.c_char_p, []),
    "sspd_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "sspd_device_ordinals": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int)]),
    "sspd_grid_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                   C.c_uint32, C.POINTER(grid_p)]),
    "sspd_grid_clone": (C.c_int, [grid_p, C.c_int, C.POINTER(grid_p)]),
    "sspd_grid_destroy": (C.c_int, [grid_p]),
    "sspd_grid_info": (C.c_int, [grid_p, u64p, C.POINTER(C.c_int), u32p]),
    "sspd_grid_create_narrow": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                          C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(grid_p)]),
    "sspd_grid_stamp_width": (C.c_int, [grid_p, u32p, u32p]),
    "sspd_grid_create_sharded": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                           C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(grid_p)]),
    "sspd_grid_owned": (C.c_int, [grid_p, u64p, u64p]),
    "sspd_reconstruct_async": (C.c_int, [grid_p, C.c_uint32, C.c_uint64, C.c_uint64]),
    "sspd_reconstruct_collect": (C.c_int, [grid_p, C.POINTER(Detection_t), C.c_uint64, u64p, u32p, u64p]),
    "sspd_set_shard": (C.c_int, [grid_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64]),
    "sspd_set_shard_relay": (C.c_int, [grid_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64]),
    "sspd_shard_relay": (C.c_int, [grid_p, C.c_void_p, C.c_uint64]),
    "sspd_shard_relay_regions": (C.c_int, [grid_p, C.c_void_p, C.c_uint64, u64p, C.c_uint32]),
    "sspd_shard_sent": (C.c_int, [grid_p, C.POINTER(C.c_void_p)]),
    "sspd_shard_receive": (C.c_int, [grid_p, C.c_void_p, C.c_uint64]),
    "sspd_shard_relay_regions_dev": (C.c_int, [grid_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint32]),
    "sspd_shard_receive_regions_dev": (C.c_int, [grid_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                                 C.c_uint32, C.c_uint32]),
    "sspd_shard_overflow": (C.c_int, [grid_p, C.POINTER(C.c_int)]),
    "sspd_reduce_words": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.c_uint32, C.c_uint64, C.c_int, C.c_void_p,
                                    C.c_void_p]),
    "sspd_shard_hot": (C.c_int, [grid_p, C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p), u64p]),
    "sspd_shard_select": (C.c_int, [grid_p, C.c_uint32, C.c_uint64, C.c_uint64, u64p, C.POINTER(C.c_void_p), u64p,
                                    u32p, u64p]),
    "sspd_shard_finish": (C.c_int, [grid_p, C.c_uint64, C.POINTER(Detection_t), C.c_uint64, u64p]),
    "sspd_grid_set_stream": (C.c_int, [grid_p, C.c_void_p]),
    "sspd_grid_stream": (C.c_int, [grid_p, C.POINTER(C.c_void_p)]),
    "sspd_scan_records": (C.c_int, [grid_p, C.c_void_p, C.c_uint64, C.c_int]),
    "sspd_device_alloc": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]),
    "sspd_device_free": (C.c_int, [C.c_int, C.c_void_p]),
    "sspd_release_cached": (C.c_int, [C.c_int, C.POINTER(C.c_uint64)]),
    "sspd_enable_peer_access": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "sspd_grid_copy": (C.c_int, [grid_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int]),
    "sspd_grid_synchronize": (C.c_int, [grid_p]),
    "sspd_scan": (C.c_int, [grid_p, C.c_void_p, C.c_uint64, C.c_int]),
    "sspd_advance": (C.c_int, [grid_p, C.c_uint32]),
    "sspd_get_distances": (C.c_int, [grid_p, u16p, C.c_uint64, C.c_uint64]),
    "sspd_put_distances": (C.c_int, [grid_p, u16p, C.c_uint64, C.c_uint64]),
    "sspd_active_counts": (C.c_int, [grid_p, C.c_uint32, u32p]),
    "sspd_hot_sets": (C.c_int, [grid_p, C.c_uint32, C.c_uint64, u32p, u32p]),
    "sspd_finalize": (C.c_int, [grid_p, u32p, C.c_uint64, C.c_uint32, C.c_uint64, u8p, u32p,
                                u32p]),
    "sspd_reconstruct": (C.c_int, [grid_p, C.c_uint32, C.c_uint64, C.c_uint64,
                                   C.POINTER(Detection_t), C.c_uint64, u64p, u32p, u64p]),
    "sspd_merge": (C.c_int, [C.POINTER(grid_p), C.c_uint64, C.c_int, grid_p]),
    "sspd_equal": (C.c_int, [grid_p, grid_p, C.POINTER(C.c_int)]),
    "sspd_track_window": (C.c_int, [grid_p, C.c_uint32]),
    "sspd_grid_stamps": (C.c_int, [grid_p, C.POINTER(C.c_void_p), u64p]),
    "sspd_grid_touched": (C.c_int, [grid_p, C.POINTER(C.c_void_p), u64p]),
    "sspd_commit": (C.c_int, [grid_p]),
    "sspd_set_exchange": (C.c_int, [grid_p, C.c_int]),
    "sspd_grid_new_pairs": (C.c_int, [grid_p, C.POINTER(C.c_void_p), u64p]),
    "sspd_set_push": (C.c_int, [grid_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64]),
    "sspd_scan_mode": (C.c_int, [grid_p, C.c_int, C.c_int]),
    "sspd_grid_fresh_pairs": (C.c_int, [grid_p, u64p]),
    "sspd_grid_keyset": (C.c_int, [grid_p, C.POINTER(C.c_void_p), u32p]),
    "sspd_checked_status": (C.c_int, [C.c_int, u32p, u64p, C.c_int]),
    "sspd_profile_enable": (C.c_int, [grid_p, C.c_int]),
    "sspd_profile_read": (C.c_int, [grid_p, C.c_char_p, C.POINTER(C.c_double), u64p, u64p]),
    "sspd_profile_reset": (C.c_int, [grid_p]),
    "sspd_launch_count": (C.c_uint64, []),
    "sspd_grid_io_bytes": (C.c_int, [grid_p, u64p, u64p, C.c_int]),
    "sspd_synth_zipf_cdf": (C.c_int, [C.c_uint32, C.c_double, C.c_void_p]),
    "sspd_synth_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                  C.c_void_p]),
    "sspd_synth_device": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                    C.c_uint64, C.c_void_p, C.c_void_p]),
    "sspd_synth_super_cip": (C.c_uint32, [C.c_void_p, C.c_uint32]),
    "sspd_exact_counts": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), u64p, C.c_uint32, C.c_uint64,
                                    C.c_uint32, u32p, u32p, C.c_uint64, u64p, C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library (no GPU work happens at load time)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (the B200 path has no CPU fallback)")
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SspdError(RuntimeError):
    pass


class InvalidArgument(SspdError, ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(SspdError, IndexError):
    """std::out_of_range in the reference."""


class CandidateOverflow(SspdError):
    """sspd::CandidateOverflow (rsea.hpp:38-43)."""

    def __init__(self, msg: str, level: int, count: int):
        super().__init__(msg)
        self.level = level
        self.count = count


class CudaError(SspdError):
    pass


class NoDevice(SspdError):
    pass


_EXC = {SSPD_INVALID_ARGUMENT: InvalidArgument, SSPD_OUT_OF_RANGE: OutOfRange,
        SSPD_CUDA_ERROR: CudaError, SSPD_NO_DEVICE: NoDevice}


def check(status: int):
    if status == SSPD_OK:
        return
    msg = load().sspd_last_error().decode()
    raise _EXC.get(status, SspdError)(msg)
