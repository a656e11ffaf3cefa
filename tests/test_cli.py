"""The `sspd` command line (paper_1803_11036_b200/bin/sspd), checked the way
the reference's tests/cli_test.sh checks the reference CLI: deterministic
synth, oracle == generator truth, detect finds the planted hosts every slot,
reports byte-identical across --workers and --strategy, eval row counts,
snapshot info/merge idempotence, incompatible-q message, exit codes 2 and 3.
With oracle/_ref present, detect's report also equals the compiled
reference's run_detection printed the same way (slot,ip,estimate with the
default 6-significant-digit formatting, sspd.cpp:102-108)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SSPD = os.path.join(ROOT, "paper_1803_11036_b200", "bin", "sspd")
SPEC = """slots 6
background hosts=100 zipf=1.1 pairs-per-slot=300 max-distinct=8
super cip=10.0.0.1 count=256 from=0 to=5
super cip=10.0.0.2 count=300 from=0 to=5
"""


def run(*args, check=True):
    p = subprocess.run([SSPD, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check and p.returncode != 0:
        raise AssertionError(f"sspd {args} -> {p.returncode}: {p.stderr}")
    return p


@pytest.fixture()
def work(tmp_path):
    if not os.path.exists(SSPD):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1803_11036_b200", "csrc")],
                       check=True, capture_output=True)
    spec = tmp_path / "spec.txt"
    spec.write_text(SPEC)
    run("synth", spec, "--desk", "--k", 5, "--seed", "5eed", "-o", tmp_path / "trace.bin",
        "--truth-out", tmp_path / "truth.csv")
    return tmp_path


def test_synth_deterministic_and_oracle_matches(work):
    run("synth", work / "spec.txt", "--desk", "--k", 5, "--seed", "5eed", "-o", work / "t2.bin",
        "--truth-out", work / "truth2.csv")
    assert (work / "trace.bin").read_bytes() == (work / "t2.bin").read_bytes()
    assert (work / "truth.csv").read_bytes() == (work / "truth2.csv").read_bytes()
    run("synth", work / "spec.txt", "--desk", "--k", 5, "--seed", "5eed", "--format", "text",
        "-o", work / "trace.txt")
    assert ",10.0.0.1," in (work / "trace.txt").read_text()
    run("oracle", work / "trace.bin", "--desk", "--k", 5, "-o", work / "truth_oracle.csv")
    assert (work / "truth.csv").read_bytes() == (work / "truth_oracle.csv").read_bytes()


def test_eval_rows(work):
    rows = [f"{s},10.0.0.1,300" for s in range(6)]
    (work / "reports.csv").write_text("\n".join(rows) + "\n")
    run("eval", "--reports", work / "reports.csv", "--truth", work / "truth.csv", "--theta", 128,
        "-o", work / "eval.csv")
    lines = (work / "eval.csv").read_text().splitlines()
    assert len(lines) == 7 and sum(line.startswith("mean,") for line in lines) == 1


def test_exit_codes(work):
    p = run("detect", work / "trace.bin", "--eta", 256, "--q", 8, "--delta", 6, "--r", 5,
            "--theta", 128, "-o", os.devnull, check=False)
    assert p.returncode == 2 and "coverage" in p.stderr
    p = run("detect", work / "does-not-exist", "--desk", "-o", os.devnull, check=False)
    assert p.returncode == 3


def test_detect_shard_errors_in_argument_order(work):
    """Shard files load concurrently; the first bad file named is the one reported."""
    good = (work / "trace.bin").read_bytes()
    (work / "trunc.bin").write_bytes(good[:8 + 12 * 3 + 5])
    (work / "magic.bin").write_bytes(b"XXXX" + good[4:])
    p = run("detect", work / "trace.bin", work / "trunc.bin", work / "magic.bin", work / "missing.bin",
            "--desk", "-o", os.devnull, check=False)
    assert p.returncode == 3 and "truncated record at position 3" in p.stderr, p.stderr
    p = run("detect", work / "magic.bin", work / "trunc.bin", "--desk", "-o", os.devnull, check=False)
    assert p.returncode == 3 and "bad magic" in p.stderr and "truncated" not in p.stderr, p.stderr
    p = run("detect", work / "trace.bin", work / "missing.bin", work / "trunc.bin", "--desk",
            "-o", os.devnull, check=False)
    assert p.returncode == 3 and "missing.bin" in p.stderr, p.stderr


@pytest.mark.gpu
def test_detect_and_snapshots(gpu, work):
    run("detect", work / "trace.bin", "--desk", "--k", 5, "--seed", "5eed", "-o", work / "r.csv")
    text = (work / "r.csv").read_text()
    for slot in range(6):
        assert f"\n{slot},10.0.0.1," in "\n" + text
        assert f"\n{slot},10.0.0.2," in "\n" + text
    run("detect", work / "trace.bin", "--desk", "--k", 5, "--seed", "5eed", "--workers", 8,
        "-o", work / "r8.csv")
    run("detect", work / "trace.bin", "--desk", "--k", 5, "--seed", "5eed", "--strategy",
        "recursive", "-o", work / "rr.csv")
    assert (work / "r8.csv").read_bytes() == (work / "r.csv").read_bytes()
    assert (work / "rr.csv").read_bytes() == (work / "r.csv").read_bytes()
    for bits in (8, 16):  # narrow-stamp grids (B200 extension): byte-identical reports
        run("detect", work / "trace.bin", "--desk", "--k", 5, "--seed", "5eed", "--stamp-width", bits,
            "-o", work / f"rw{bits}.csv")
        assert (work / f"rw{bits}.csv").read_bytes() == (work / "r.csv").read_bytes()
    p = run("detect", work / "trace.bin", "--desk", "--k", 5, "--stamp-width", 12, "-o", os.devnull,
            check=False)
    assert p.returncode == 2 and "stamp width" in p.stderr

    run("snapshot", "export", work / "trace.bin", "--desk", "--k", 5, "--seed", "5eed",
        "-o", work / "s1")
    info = run("snapshot", "info", work / "s1").stdout
    assert "eta=256" in info and "slot=5" in info
    run("snapshot", "merge", work / "s1", work / "s1", "-o", work / "sm")
    assert (work / "s1").read_bytes() == (work / "sm").read_bytes()
    run("snapshot", "merge", work / "s1", work / "s1", "--merge-policy", "paper-max",
        "-o", work / "smx")
    assert (work / "s1").read_bytes() == (work / "smx").read_bytes()
    run("snapshot", "export", work / "trace.bin", "--k", 5, "--seed", "5eed", "--eta", 256,
        "--q", 11, "--delta", 8, "--r", 5, "--theta", 128, "-o", work / "s2")
    p = run("snapshot", "merge", work / "s1", work / "s2", "-o", os.devnull, check=False)
    assert p.returncode != 0 and "q=10" in p.stderr and "q=11" in p.stderr

    # the exported grid is the oracle's after the same scans/advances
    trace = np.fromfile(work / "trace.bin", dtype=np.uint32)[2:].reshape(-1, 3)
    o = O.OracleGrid(q=10, r=5, delta=8, seed=0x5eed, eta=256)
    slots = trace[:, 0]
    for s in range(int(slots.max()) + 1):
        o.scan(trace[slots == s][:, 1:])
        if s < slots.max():
            o.advance()
    payload = np.frombuffer((work / "s1").read_bytes()[56:], dtype="<u2")
    assert np.array_equal(payload, o.cells())

    if O.ref_available():
        nrep, rows = O.ref_run_detection([trace], q=10, r=5, delta=8, seed=0x5eed, eta=256,
                                         k=5, theta=128.0)
        want = "".join(f"{s},{d.cip >> 24}.{d.cip >> 16 & 255}.{d.cip >> 8 & 255}.{d.cip & 255},"
                       f"{d.estimate:.6g}\n" for s, d in rows)
        assert text == want

    # three router shards, loaded concurrently: union-min merging gives the single-trace grid,
    # so the reports are byte-identical to the one-file run (and to the reference's pipeline)
    head = (work / "trace.bin").read_bytes()[:8]
    shard_paths = []
    for i in range(3):
        path = work / f"shard{i}.bin"
        path.write_bytes(head + np.ascontiguousarray(trace[i::3]).astype("<u4").tobytes())
        shard_paths.append(path)
    run("detect", *shard_paths, "--desk", "--k", 5, "--seed", "5eed", "-o", work / "r3.csv")
    assert (work / "r3.csv").read_bytes() == (work / "r.csv").read_bytes()
    if O.ref_available():
        nrep, rows = O.ref_run_detection([trace[i::3] for i in range(3)], q=10, r=5, delta=8,
                                         seed=0x5eed, eta=256, k=5, theta=128.0)
        want3 = "".join(f"{s},{d.cip >> 24}.{d.cip >> 16 & 255}.{d.cip >> 8 & 255}.{d.cip & 255},"
                        f"{d.estimate:.6g}\n" for s, d in rows)
        assert (work / "r3.csv").read_text() == want3


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("q,r,delta,eta,k,theta", [
    (14, 5, 0, 2048, 5, 1024), (14, 2, 0, 1, 0, 0.5), (8, 5, 6, 256, 5, 128), (17, 3, 17, 2048, 65535, 1024)])
def test_invalid_configuration_message_equals_reference(work, q, r, delta, eta, k, theta):
    """`sspd detect` prints validate_config's whole list (sspd.cpp:65-70, 401-406),
    byte for byte the reference's messages, and exits 2 -- delta=0 included
    (hashing.cpp:74-78 reports the coverage rule for it too)."""
    p = run("detect", work / "trace.bin", "--q", q, "--r", r, "--delta", delta, "--eta", eta,
            "--k", k, "--theta", theta, "-o", os.devnull, check=False)
    want = "error: invalid configuration:" + "".join(
        "\n  " + m for m in O.ref_validate_all(q, r, delta, eta, k, theta)) + "\n"
    assert p.returncode == 2
    assert p.stderr == want


@pytest.mark.gpu
def test_detect_devices_option_matches_one_router(gpu, work):
    """`sspd detect --devices N` runs N routers (partial grids, relays, peer
    reduces; several share a GPU when the box has fewer) and prints the
    one-router report byte for byte; --devices 0 is a usage error."""
    run("detect", work / "trace.bin", "--desk", "--k", 5, "--seed", "5eed", "-o", work / "r1.csv")
    for n in (2, 3):
        run("detect", work / "trace.bin", "--desk", "--k", 5, "--seed", "5eed", "--devices", n,
            "-o", work / f"r{n}.csv")
        assert (work / f"r{n}.csv").read_bytes() == (work / "r1.csv").read_bytes()
    p = run("detect", work / "trace.bin", "--desk", "--devices", 0, "-o", os.devnull, check=False)
    assert p.returncode == 1
