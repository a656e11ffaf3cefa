"""The reference's OWN tests, unchanged, against the drop-in.

tests/refsuite/Makefile compiles /root/reference/proj/tests/{acceptance,
test_hashing, test_estimator, test_rsea, test_snapshot, test_workload,
test_pipeline}.cpp as they lie -- against include/sspd/*.hpp and
libsspd.so (the B200 library), with tests/refsuite/doctest.h standing in for
the doctest the reference never vendored -- and stages cli_test.sh beside
them.  The binaries travel to the GPU box, where /root/reference does not
exist.  This is the proof that reference callers "compile unchanged"
(ref tests/CMakeLists.txt:1-13).

The host-only suites (hashing, estimator, workload) run here on CPU; the
ones that build grids need the B200.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "refsuite", "bin")
SSPD = os.path.join(ROOT, "paper_1803_11036_b200", "bin", "sspd")


def _bin(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "refsuite")], check=True,
                       capture_output=True)
    if not os.path.exists(path):
        pytest.skip(f"{name}: the reference's test sources were not available to build it")
    return path


def _doctest(name, timeout):
    p = subprocess.run([_bin(name)], capture_output=True, text=True, timeout=timeout)
    out = p.stdout + p.stderr
    tail = "\n".join(out.strip().splitlines()[-30:])
    assert p.returncode == 0, tail
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| 0 failed", p.stdout)
    assert m and m.group(1) == m.group(2) and int(m.group(1)) > 0, tail
    return out


@pytest.mark.parametrize("suite", ["hashing", "estimator", "workload"])
def test_reference_host_suite(suite):
    _doctest(f"test_{suite}", 600)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["rsea", "snapshot", "pipeline"])
def test_reference_device_suite(gpu, suite):
    _doctest(f"test_{suite}", 900)


@pytest.mark.gpu
def test_reference_acceptance_all_criteria(gpu):
    """acceptance.cpp:387-415, all 10 criteria, with criterion 9's full-size
    snapshot export enabled (SSPD_BIG_MEM=1)."""
    env = dict(os.environ, SSPD_BIG_MEM="1")
    p = subprocess.run([_bin("sspd_acceptance")], capture_output=True, text=True, timeout=1800,
                       env=env)
    print(p.stdout)
    passed = re.findall(r"^criterion .*: PASS", p.stdout, re.M)
    assert p.returncode == 0, p.stdout + p.stderr[-3000:]
    assert len(passed) == 10, p.stdout


@pytest.mark.gpu
def test_reference_cli_script(gpu):
    """cli_test.sh:1-93 against bin/sspd: deterministic synth, oracle == truth,
    detect finds the planted supers every slot, byte-identical reports across
    --workers and --strategy, eval rows, snapshot info/merge, the q mismatch
    message, exit codes 2 and 3."""
    script = _bin("cli_test.sh")
    p = subprocess.run(["sh", script, SSPD], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "cli_test: all checks passed" in p.stdout
