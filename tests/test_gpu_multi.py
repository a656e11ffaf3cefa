"""The router exchanges across REAL GPUs (pipeline.cpp:76-85).

Skipped on a one-GPU box (every round-1/2 box had one); on a multi-GPU node
these run every exchange of dist.py end to end under torchrun with NCCL and
NVLink peer memory -- SHARD (partial grids, device-counted relays, peer
reduce), PUSH (P2P stores during the scan), PAIRS, BITMAP and the literal
all-reduce(max) of the stamps -- each rank checking reports and cells
against the oracle's union-min merge (tests/dist_worker.py), and the C++
multi-router run_detection (`sspd detect --devices N`) against one GPU.
"""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SSPD = os.path.join(ROOT, "paper_1803_11036_b200", "bin", "sspd")

pytestmark = pytest.mark.gpu


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


needs2 = pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs (this box has fewer)")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@needs2
@pytest.mark.parametrize("merge", ["shard", "push", "pairs", "bitmap", "stamps"])
def test_router_exchange_across_gpus(gpu, merge):
    n = min(_gpus(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "dist_worker.py"), "--merge", merge]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "dist_worker ok" in p.stdout


@needs2
def test_cli_detect_devices_matches_one_gpu(gpu, tmp_path):
    """`sspd detect --devices N` (one router per GPU, partial grids, NVLink
    relays and peer reduces in one process) prints the one-GPU report."""
    spec = tmp_path / "spec.txt"
    spec.write_text("slots 6\nbackground hosts=2000 zipf=1.1 pairs-per-slot=20000 max-distinct=8\n"
                    "super cip=10.0.0.1 count=300 from=0 to=5\nsuper cip=10.0.0.2 count=400 from=1 to=5\n")
    run = lambda *a: subprocess.run([SSPD, *map(str, a)], capture_output=True, text=True, timeout=600)  # noqa: E731
    assert run("synth", spec, "--desk", "--k", 5, "--seed", "5eed", "-o", tmp_path / "t.bin").returncode == 0
    one = run("detect", tmp_path / "t.bin", "--desk", "--k", 5, "--seed", "5eed", "-o", tmp_path / "r1.csv")
    many = run("detect", tmp_path / "t.bin", "--desk", "--k", 5, "--seed", "5eed", "--devices", min(_gpus(), 8),
               "-o", tmp_path / "rn.csv")
    assert one.returncode == 0 and many.returncode == 0, one.stderr + many.stderr
    assert (tmp_path / "r1.csv").read_bytes() == (tmp_path / "rn.csv").read_bytes()
    assert "10.0.0.1" in (tmp_path / "r1.csv").read_text()
