"""Trace files (workload.hpp:26-32, workload.cpp read_trace/write_trace) as
numpy (n, 3) uint32 arrays of (ts, cip, oip) -- the records
run_detection and Grid.scan_records take.

Binary: "SSPT", u32 LE version 1, then 12-byte LE records.  Text: one
"ts,a.b.c.d,a.b.c.d" line per record, '#' comments and blank lines skipped.
Errors carry the reference's messages (RuntimeError, as std::runtime_error).
"""
from __future__ import annotations

import io
import os
import re

import numpy as np

MAGIC = b"SSPT"
VERSION = 1


def _check_order(ts: np.ndarray) -> None:
    if len(ts) > 1:
        bad = np.flatnonzero(ts[1:] < ts[:-1])
        if len(bad):
            raise RuntimeError(f"trace: timestamp regression at record {int(bad[0]) + 1}")


_WS = " \t\n\v\f\r"


def _sto_prefix(s: str) -> tuple[int, int]:
    """std::stoi/stoull: leading whitespace, a sign, then the longest digit run."""
    m = re.match(f"[{_WS}]*([+-]?[0-9]+)", s)
    if not m:
        raise ValueError(s)
    return int(m.group(1)), m.end()


def _parse_ipv4(text: str) -> int:
    """parse_ipv4 (workload.cpp): a plain integer, or a dotted quad whose
    octets are read like std::stoi."""
    if "." not in text:
        v, used = _sto_prefix(text)
        if used != len(text) or not 0 <= v <= 0xFFFFFFFF:
            raise ValueError(text)
        return v
    parts = text.split(".")
    if parts and parts[-1] == "":  # getline drops the field after a trailing '.'
        parts.pop()
    if len(parts) != 4:
        raise ValueError(text)
    ip = 0
    for part in parts:
        if not part or len(part) > 3:
            raise ValueError(text)
        v, _ = _sto_prefix(part)
        if not 0 <= v <= 255:
            raise ValueError(text)
        ip = ip << 8 | v
    return ip


def _format_ipv4(ip: int) -> str:
    return f"{ip >> 24}.{ip >> 16 & 255}.{ip >> 8 & 255}.{ip & 255}"


def read_trace(src, fmt: str = "binary", mmap: bool = False) -> np.ndarray:
    """src: a path or a binary file object.  mmap=True (a binary trace at a
    path): a read-only memory map of the records, checked like a read, so
    that run_detection / Grid.scan_records pack slot runs straight from the
    page cache into pinned staging, with no copy of the whole trace."""
    if isinstance(src, (str, os.PathLike)):
        if mmap and fmt == "binary":
            size = os.path.getsize(src)
            with open(src, "rb") as f:
                head = f.read(8)
            if size == 0:
                return np.zeros((0, 3), np.uint32)
            if len(head) < 8 or head[:4] != MAGIC:
                raise RuntimeError("trace: bad magic")
            if int.from_bytes(head[4:8], "little") != VERSION:
                raise RuntimeError("trace: unsupported version")
            whole = (size - 8) // 12
            if whole == 0:
                if size > 8:
                    raise RuntimeError("trace: truncated record at position 0")
                return np.zeros((0, 3), np.uint32)
            recs = np.memmap(src, dtype="<u4", mode="r", offset=8, shape=(whole, 3))
            _check_order(recs[:, 0])
            if (size - 8) % 12:
                raise RuntimeError(f"trace: truncated record at position {whole}")
            return recs
        with open(src, "rb") as f:
            return read_trace(f, fmt)
    if fmt == "binary":
        data = src.read()
        if not data:
            return np.zeros((0, 3), np.uint32)
        if len(data) < 8 or data[:4] != MAGIC:
            raise RuntimeError("trace: bad magic")
        if int.from_bytes(data[4:8], "little") != VERSION:
            raise RuntimeError("trace: unsupported version")
        body = len(data) - 8
        whole = body // 12
        recs = np.frombuffer(data, dtype="<u4", count=whole * 3, offset=8).reshape(whole, 3)
        _check_order(recs[:, 0])  # the reference reports a regression before a truncation
        if body % 12:
            raise RuntimeError(f"trace: truncated record at position {whole}")
        return recs.astype(np.uint32)
    if fmt != "text":
        raise ValueError(f"unknown trace format {fmt!r}")
    text = src.read()
    if isinstance(text, bytes):
        text = text.decode("latin-1")
    rows = []
    last = None
    for lineno, line in enumerate(io.StringIO(text), 1):
        line = line[:-1] if line.endswith("\n") else line
        if not line or line.startswith("#"):
            continue
        f = line.split(",", 2)
        try:
            if len(f) != 3:
                raise ValueError(line)
            ts, _ = _sto_prefix(f[0])  # std::stoull, then the cast to u32
            if not -2**64 < ts < 2**64:
                raise ValueError(line)
            rec = ((ts % 2**64) & 0xFFFFFFFF, _parse_ipv4(f[1]), _parse_ipv4(f[2]))
        except ValueError:
            raise RuntimeError(f"trace: malformed line {lineno}") from None
        if last is not None and rec[0] < last:
            raise RuntimeError(f"trace: timestamp regression at record {len(rows)}")
        last = rec[0]
        rows.append(rec)
    return np.array(rows, dtype=np.uint32).reshape(-1, 3)


def write_trace(records, dst, fmt: str = "binary") -> None:
    """records: (n, 3) (ts, cip, oip); dst: a path or a binary file object."""
    if isinstance(dst, (str, os.PathLike)):
        with open(dst, "wb") as f:
            return write_trace(records, f, fmt)
    r = np.ascontiguousarray(records, dtype=np.uint32).reshape(-1, 3)
    if fmt == "binary":
        dst.write(MAGIC + VERSION.to_bytes(4, "little"))
        dst.write(r.astype("<u4").tobytes())
        return
    if fmt != "text":
        raise ValueError(f"unknown trace format {fmt!r}")
    dst.write("".join(f"{int(t)},{_format_ipv4(int(c))},{_format_ipv4(int(o))}\n" for t, c, o in r).encode())
