"""The drop-in boundary loads without a GPU and exports what it declares."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_1803_11036_b200 as P
from paper_1803_11036_b200 import _cabi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sspd_cuda.h")
LIBDIR = os.path.join(ROOT, "paper_1803_11036_b200", "lib")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sspd_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("sspd_grid_create", "sspd_scan", "sspd_advance", "sspd_hot_sets",
                 "sspd_reconstruct", "sspd_merge", "sspd_get_distances"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_cabi.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python bindings cover the whole header
    assert set(declared()) <= set(_cabi.SIGNATURES), set(declared()) - set(_cabi.SIGNATURES)


def test_cxx_api_library_exports_the_reference_surface():
    out = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(LIBDIR, "libsspd.so")],
                         capture_output=True, text=True, check=True).stdout
    for sym in ("sspd::Rsea::scan_batch", "sspd::Rsea::advance_slot", "sspd::Rsea::hot_sets",
                "sspd::Rsea::reconstruct_leveled", "sspd::Rsea::reconstruct_recursive",
                "sspd::Rsea::finalize_candidate", "sspd::merge_rseas", "sspd::run_detection",
                "sspd::export_snapshot", "sspd::import_snapshot", "sspd::synth_trace",
                "sspd::exact_counts", "sspd::read_trace", "sspd::validate_config",
                "sspd::hot_cutoff", "sspd::estimate_cardinality"):
        assert sym in out, sym


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", _cabi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    """Without a usable device the product path fails loudly."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    with pytest.raises(P.SspdError):
        P.Grid(q=10, r=5, delta=8, eta=256)
    assert P.hot_cutoff(2048, 1024) == 806
