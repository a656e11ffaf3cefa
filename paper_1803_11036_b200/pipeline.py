"""run_detection over device grids, in Python (reference: proj/src/pipeline.cpp:16-89;
the C++ drop-in is csrc/host/pipeline.cpp).

Per slot: scan every shard's pairs of the slot, merge (union-min on one grid,
which equals the reference's merged copy because the merge is idempotent and
commutes with advance_slot; paper-max on per-node grids merged into a scratch
grid), reconstruct on the merged grid, advance.  Reports are
(slot, [Detection...]) with the reference's dedup and ordering.
"""
from __future__ import annotations

import numpy as np

from ._cabi import InvalidArgument, PAPER_MAX, UNION_MIN
from .grid import Grid, merge_rseas


def validate_config(q: int, r: int, delta: int, eta: int, k: int, theta: float) -> list[str]:
    """validate_config (hashing.cpp:63-87), same diagnostics."""
    out = []
    if q < 1 or q > 16:
        out.append(f"q must be in [1, 16], got {q}")
    if delta == 0 or delta >= q:
        out.append(f"delta must satisfy 0 < delta < q, got delta={delta} q={q}")
    if r < 3:
        out.append(f"r must be >= 3, got {r}")
    if r >= 3 and delta < q and (r - 2) * delta + q < 32:
        out.append(f"address coverage (r-2)*delta+q = {(r - 2) * delta + q} < 32")
    if eta < 2:
        out.append(f"eta must be >= 2, got {eta}")
    if k < 1 or k > 65534:
        out.append(f"k must be in [1, 65534], got {k}")
    if theta < 1:
        out.append(f"theta must be >= 1, got {theta:f}")
    return out


def run_detection(shards, q=14, r=5, delta=6, seed=0, eta=2048, mu=1.0, k=300, start=0,
                  theta=1024.0, policy=UNION_MIN, recursive=False, candidate_cap=1 << 24,
                  device=0, probe=None):
    """shards: list of (n, 3) uint32 arrays of (ts, cip, oip) records, time sorted.
    probe(slot, grid) sees the grid reconstruction runs on, per slot."""
    if not len(shards):
        raise InvalidArgument("run_detection: no trace shards")
    problems = validate_config(q, r, delta, eta, k, theta)
    if problems:
        raise InvalidArgument("run_detection: " + problems[0])
    shards = [np.ascontiguousarray(s, dtype=np.uint32).reshape(-1, 3) for s in shards]
    n_slots = 0
    slot_of = []
    for s in shards:
        if len(s) and int(s[:, 0].min()) < start:
            raise InvalidArgument("run_detection: record before start")
        so = ((s[:, 0].astype(np.float64) - start) / mu).astype(np.uint64)  # slot_of, workload.hpp:64-66
        slot_of.append(so)
        if len(so):
            n_slots = max(n_slots, int(so.max()) + 1)
    union = policy == UNION_MIN or len(shards) == 1
    nodes = [Grid(q, r, delta, seed, eta, device=device) for _ in range(1 if union else len(shards))]
    for g in nodes:
        g.candidate_cap = candidate_cap
        g.track_window(k)
    reports = []
    # union-min + leveled pipelines like the C++ run_detection: a slot's
    # reconstruction is queued and collected after the next slot's scan
    pipelined = union and not recursive and candidate_cap <= (1 << 26)
    pending = None
    # time-sorted shards: each slot is a contiguous run of records, scanned
    # where it lies (sspd_scan_records); otherwise select the slot's records
    ordered = all(len(so) < 2 or bool(np.all(so[1:] >= so[:-1])) for so in slot_of)
    bounds = [np.searchsorted(so, np.arange(n_slots + 1, dtype=np.uint64)) if ordered else None
              for so in slot_of]
    for slot in range(n_slots):
        if ordered:
            parts = [s[b[slot]:b[slot + 1]] for s, b in zip(shards, bounds)]
        else:
            parts = [s[so == slot] for s, so in zip(shards, slot_of)]
        if union:
            for p in parts:
                if len(p):
                    nodes[0].scan_records(p)
            target = nodes[0]
        else:
            for g, p in zip(nodes, parts):
                if len(p):
                    g.scan_records(p)
            target = merge_rseas(nodes, PAPER_MAX)
            target.candidate_cap = candidate_cap
        if pending is not None:
            reports.append((pending, target.reconstruct_collect()))
            pending = None
        if probe is not None:
            probe(slot, target)
        if pipelined:
            target.reconstruct_async(k, theta)
            pending = slot
        else:
            dets = (target.reconstruct_recursive(k, theta) if recursive
                    else target.reconstruct_leveled(k, theta))
            reports.append((slot, dets))
        for g in nodes:
            g.advance_slot()
    if pending is not None:
        reports.append((pending, nodes[0].reconstruct_collect()))
    return reports
