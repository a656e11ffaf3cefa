"""Run the C++ API test binaries (tests/cpp, built by __graft_entry__.build()).

test_api_host exercises the host-only parts of the drop-in API (no GPU);
test_api_gpu exercises sspd::Rsea / merge_rseas / snapshots / run_detection
on the device, with differential checks against the compiled reference when
it was linked in.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin")


def _binary(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp")], check=True,
                       capture_output=True)
    return path


def _run(name, timeout):
    p = subprocess.run([_binary(name)], capture_output=True, text=True, timeout=timeout)
    tail = "\n".join(p.stderr.strip().splitlines()[-25:])
    assert p.returncode == 0, tail
    assert "0 checks failed" in p.stderr, tail


def test_cpp_host_api():
    _run("test_api_host", 300)


@pytest.mark.gpu
def test_cpp_device_api(gpu):
    _run("test_api_gpu", 900)
