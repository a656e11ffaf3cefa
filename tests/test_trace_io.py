"""Python trace I/O (paper_1803_11036_b200/trace.py) against the C++ drop-in's
read_trace/write_trace (workload.cpp, through `sspd synth`): same bytes
written, same records read, the reference's error messages and positions
(test_api_host.cpp "trace I/O round trips and errors")."""
import io

import numpy as np
import pytest

from paper_1803_11036_b200 import trace as T
from test_cli import run, work  # noqa: F401  (the fixture)


def test_cli_traces_round_trip(work):  # noqa: F811
    run("synth", work / "spec.txt", "--desk", "--k", 5, "--seed", "5eed", "--format", "text",
        "-o", work / "trace.txt")
    binary = T.read_trace(work / "trace.bin")
    text = T.read_trace(work / "trace.txt", "text")
    mapped = T.read_trace(work / "trace.bin", mmap=True)
    assert binary.shape[1] == 3 and len(binary) > 1000
    assert np.array_equal(binary, text) and np.array_equal(binary, mapped)
    data = (work / "trace.bin").read_bytes()
    (work / "cut.bin").write_bytes(data[:-7])
    with pytest.raises(RuntimeError, match=f"truncated record at position {len(binary) - 1}"):
        T.read_trace(work / "cut.bin", mmap=True)
    for fmt, name in [("binary", "trace.bin"), ("text", "trace.txt")]:
        out = io.BytesIO()
        T.write_trace(binary, out, fmt)
        assert out.getvalue() == (work / name).read_bytes(), fmt


def test_errors_and_edge_cases():
    recs = np.array([[0, 1, 2], [0, 0xC0A80101, 0x08080808], [5, 7, 9]], np.uint32)
    for fmt in ("binary", "text"):
        b = io.BytesIO()
        T.write_trace(recs, b, fmt)
        assert np.array_equal(T.read_trace(io.BytesIO(b.getvalue()), fmt), recs)
    assert T.read_trace(io.BytesIO(b"")).shape == (0, 3)
    with pytest.raises(RuntimeError, match="bad magic"):
        T.read_trace(io.BytesIO(b"XXXX\x01\0\0\0"))
    with pytest.raises(RuntimeError, match="unsupported version"):
        T.read_trace(io.BytesIO(b"SSPT\x02\0\0\0"))
    with pytest.raises(RuntimeError, match="timestamp regression at record 1"):
        T.read_trace(io.BytesIO(b"5,1.2.3.4,5.6.7.8\n4,1.2.3.4,5.6.7.8\n"), "text")
    with pytest.raises(RuntimeError, match="malformed line 1"):
        T.read_trace(io.BytesIO(b"1,2\n"), "text")
    b = io.BytesIO()
    T.write_trace(recs, b)
    with pytest.raises(RuntimeError, match="truncated record at position 2"):
        T.read_trace(io.BytesIO(b.getvalue()[:-1]))
    back = recs.copy()
    back[0, 0] = 4
    back[1, 0] = 3
    b = io.BytesIO()
    T.write_trace(back, b)
    with pytest.raises(RuntimeError, match="timestamp regression at record 1"):
        T.read_trace(io.BytesIO(b.getvalue()[:-1]))  # regression reported before the truncation
    # parse_ipv4's forms: plain integers, std::stoi octets, a trailing '.', CRLF
    got = T.read_trace(io.BytesIO(b"# c\n\n7, 16909060,+1.2.3.4.\n8,1.2.3.4,8.8.8.8\r\n"), "text")
    assert got.tolist() == [[7, 16909060, 16909060], [8, 16909060, 0x08080808]]
    for bad in (b"1,1.2.3,4\n", b"1,1.2.3.256,4\n", b"1,1..2.3,4\n", b"1,4294967296,4\n", b"x,1,2\n",
                b"7,1.2.3.4.\r,1\n"):
        with pytest.raises(RuntimeError, match="malformed line 1"):
            T.read_trace(io.BytesIO(bad), "text")
