"""The GPU parity suites on the CHECKED build (lib/libsspd_cuda_checked.so:
kernels.cuh "CHECKED BUILD" -- bounds checks on every data-dependent stamp,
code and window-ring index, and the ring's no-underflow invariant).  This
pool closes compute-sanitizer, so these checks stand in for its memcheck on
the data-dependent accesses: every test of test_gpu_parity / _narrow / _fuzz / _keyset
runs on the checked kernels, and after each one (tests/conftest.py) no check
may have failed."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1803_11036_b200", "lib", "libsspd_cuda_checked.so")

pytestmark = pytest.mark.gpu


def test_checked_build_reports_itself(gpu):
    """The product library refuses checked_status (no checks compiled in)."""
    with pytest.raises(gpu.InvalidArgument, match="not a checked build"):
        gpu.checked_status(0)


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked library not built")
def test_parity_suites_on_checked_kernels(gpu):
    env = dict(os.environ, SSPD_LIB=CHECKED, SSPD_CHECKED_ASSERT="1")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu and not slow", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_narrow.py", "tests/test_gpu_fuzz.py",
                        "tests/test_gpu_keyset.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    tail = "\n".join((p.stdout + p.stderr).strip().splitlines()[-25:])
    assert p.returncode == 0, tail
    assert " passed" in p.stdout and "failed" not in p.stdout.splitlines()[-1], tail
    print(p.stdout.strip().splitlines()[-1])
