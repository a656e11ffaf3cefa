"""Generate tests/golden/ from the COMPILED REFERENCE (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile).  Run here, where the reference
exists; the outputs are committed and the tests read only them, so nothing on
the GPU box needs /root/reference.

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

SEEDS = [0, 1, 42, 0x5eed, 0x1234abcd, 0xfeed, 0xFFFFFFFFFFFFFFFF]
CFGS = [(14, 5, 6), (10, 5, 8), (16, 5, 6), (16, 8, 6), (12, 7, 4), (9, 12, 3)]


def keys():
    ks = [0, 0xFFFFFFFF, 0x08080808, 0xC0A80101, 0x01020304]
    ks += [1 << b for b in range(32)]
    rng = O.Mt64(4242)
    ks += [int(x) & 0xFFFFFFFF for x in rng.draw(200)]
    return ks


def main():
    R = O.ref()
    gold: dict = {"generator": "tests/golden/make_golden.py from oracle/_ref (compiled "
                               "/root/reference/proj sources)"}
    ks = keys()
    gold["keys"] = ks
    # TabulationHash values via HashSeeds (hashing.cpp:18-34)
    gold["hash"] = {hex(s): {"h1": [hex(R.ref_h1_raw(s, k)) for k in ks],
                             "row0": [hex(R.ref_row0_raw(s, k)) for k in ks]} for s in SEEDS}
    gold["hash_opposite"] = {
        f"{hex(s)}:{eta}": [R.ref_hash_opposite(s, k, eta) for k in ks]
        for s in (0x5eed, 42) for eta in (1, 2, 3, 256, 1000, 2048, 65536, 1 << 20)}
    # rhfg columns (hashing.cpp:36-43)
    rh = {}
    for q, r, d in CFGS:
        for s in (0x5eed, 0x1234abcd):
            cips = np.array(ks, dtype=np.uint32)
            cols = np.empty(len(ks) * r, dtype=np.uint32)
            R.ref_rhfg_cols(q, r, d, s, cips.ctypes.data_as(O.u32p), len(ks),
                            cols.ctypes.data_as(O.u32p))
            rh[f"{q},{r},{d},{hex(s)}"] = cols.reshape(-1, r).tolist()
    gold["rhfg"] = rh
    # assemble_ip (hashing.cpp:45-61): round trips plus random block tuples
    asm = []
    rng = O.Mt64(77)
    for q, r, d in CFGS:
        for i in range(300):
            if i < 150:
                cip = int(rng.next()) & 0xFFFFFFFF
                blocks = [((cip >> ((j * d) & 31)) & ((1 << q) - 1)) for j in range(r - 1)]
                if i % 3 == 0:
                    blocks[int(rng.next() % (r - 1))] ^= 1 << int(rng.next() % q)
            else:
                blocks = [int(rng.next()) & ((1 << q) - 1) for _ in range(r - 1)]
            b = np.array(blocks, dtype=np.uint32)
            ip = O.C.c_uint32()
            ok = R.ref_assemble_ip(q, r, d, b.ctypes.data_as(O.u32p), O.C.byref(ip))
            asm.append([q, r, d, blocks, ip.value if ok else None])
    gold["assemble"] = asm
    gold["blocks_consistent"] = [
        [q, r, d, lo, hi, R.ref_blocks_consistent(q, r, d, lo, hi)]
        for (q, r, d) in CFGS for (lo, hi) in [(0, 0), (0x3f00, 1), (0x3f00, 0xfc), (5, 5),
                                               (0xffff, 0xffff), (0x1234, 0x48)]]
    gold["hot_cutoff"] = [[eta, th, R.ref_hot_cutoff(eta, th)]
                          for eta in (2, 3, 256, 1000, 2048, 65536)
                          for th in (1.0, 2.5, 64.0, 128.0, 806.0, 1024.0, 4096.0, 1e6)]
    gold["estimate"] = [[eta, rk, R.ref_estimate(eta, rk).hex()]
                        for eta in (2, 256, 1000, 2048, 65536)
                        for rk in sorted({0, 1, eta // 3, eta // 2, 806 % eta, eta - 1, eta})]
    val = []
    for args in [(14, 5, 6, 2048, 300, 1024.0), (8, 5, 6, 2048, 300, 1024.0),
                 (17, 5, 6, 2048, 300, 1024.0), (14, 5, 14, 2048, 300, 1024.0),
                 (14, 2, 6, 2048, 300, 1024.0), (14, 5, 6, 1, 300, 1024.0),
                 (14, 5, 6, 2048, 0, 1024.0), (14, 5, 6, 2048, 65535, 1024.0),
                 (14, 5, 6, 2048, 300, 0.5), (0, 1, 0, 0, 0, 0.0)]:
        buf = O.C.create_string_buffer(256)
        n = R.ref_validate(*args, buf, 256)
        val.append([list(args), n, buf.value.decode()])
    gold["validate"] = val

    # Grids: scan/advance sequences, per-cell R_k, hot sets, reports.
    grids = []
    cases = [("desk", 10, 5, 8, 256, 0x5eed), ("paper", 14, 5, 6, 2048, 0x5eed),
             ("odd_eta", 12, 7, 4, 1000, 7), ("wide_r", 16, 8, 6, 64, 9)]
    for name, q, r, d, eta, seed in cases:
        g = O.RefGrid(q, r, d, seed, eta)
        rng = O.Mt64(7)
        steps = []
        for step in range(3):
            g.scan(rng.pairs(100_000), workers=4)
            c = g.cells()
            steps.append({"fnv": hex(O.fnv1a64(c)), "zeros": int((c == 0).sum()),
                          "ones": int((c == 1).sum())})
            g.advance(4)
        grids.append({"name": name, "cfg": [q, r, d, eta, hex(seed)], "mt_seed": 7,
                      "pairs_per_step": 100_000, "steps": steps})
    gold["grids"] = grids

    # Planted states (acceptance.cpp:207-231 style) -> hot sets, counts, reports.
    states = []
    rng = O.Mt64(106)
    for st in range(12):
        q, r, d, eta, seed = 10, 5, 8, 256, 0x106
        g = O.RefGrid(q, r, d, seed, eta)
        hosts = int(rng.next() % 8)
        ops = []
        for _ in range(hosts):
            cip = int(rng.next()) & 0xFFFFFFFF
            cnt = 32 + int(rng.next() % 512)
            oips = rng.draw(cnt).astype(np.uint32)
            g.scan(np.stack([np.full(cnt, cip, np.uint32), oips], 1))
            ops.append(["host", cip, cnt])
        g.scan(rng.pairs(2000))
        ops.append(["noise", 2000])
        if st % 3 == 0:
            g.advance(1)
            ops.append(["advance"])
        counts = {}
        for k in (1, 5, 30):
            cells = g.cells()
            per = (cells.reshape(-1, eta) < k).sum(axis=1).astype(np.uint32)
            counts[str(k)] = hex(O.fnv1a64(per))
        hot = [h.tolist() for h in g.hot_sets(30, 128.0)]
        rep = g.reconstruct(30, 128.0, leveled=True, workers=3)
        rec = g.reconstruct(30, 128.0, leveled=False)
        states.append({"cfg": [q, r, d, eta, hex(seed)], "ops": ops,
                       "cells_fnv": hex(O.fnv1a64(g.cells())), "counts_fnv": counts,
                       "hot": hot,
                       "leveled": [[x.cip, x.estimate.hex()] for x in rep],
                       "recursive": [[x.cip, x.estimate.hex()] for x in rec]})
    gold["states"] = {"mt_seed": 106, "list": states}

    # Candidate overflow (test_rsea.cpp:224-238).
    g = O.RefGrid(10, 5, 8, 0xfeed, 256)
    rng = O.Mt64(27)
    for _ in range(30):
        cip = int(rng.next()) & 0xFFFFFFFF
        g.scan(np.stack([np.full(256, cip, np.uint32), rng.draw(256).astype(np.uint32)], 1))
    ovf = {}
    for cap in (4, 100, 1000):
        try:
            g.reconstruct(30, 128.0, cap=cap, workers=2)
            ovf[str(cap)] = None
        except O.CandidateOverflow as e:
            ovf[str(cap)] = [e.level, e.count]
    gold["overflow"] = {"mt_seed": 27, "hosts": 30, "count": 256, "caps": ovf}

    # run_detection on a reference synth trace (test_pipeline.cpp make_workload),
    # single node and 4 shards (union-min), plus paper-max.
    planted = [[0x0A000000 + i, 256, 0, 7] for i in range(3)]
    trace = O.ref_synth_trace(planted, 200, 1.1, 500, 8, 8, 77, mu=1.0, k=5)
    shard_rng = O.Mt64(81)
    owner = shard_rng.draw(len(trace)) % 4
    shards = [trace[owner == i] for i in range(4)]
    np.savez_compressed(os.path.join(OUT, "pipeline_trace.npz"), trace=trace, owner=owner)
    pipe = {}
    for label, recs, pol in [("single", [trace], 0), ("sharded_union", shards, 0),
                             ("sharded_paper", shards, 1)]:
        nrep, rows = O.ref_run_detection(recs, q=10, r=5, delta=8, seed=0x5eed, eta=256, mu=1.0,
                                         k=5, theta=128.0, alpha=1024, policy=pol)
        pipe[label] = {"n_reports": nrep, "rows": [[s, d.cip, d.estimate.hex()] for s, d in rows]}
    gold["pipeline"] = {"cfg": "desk preset, seed 0x5eed, k=5, theta=128, alpha=1024",
                        "trace": "pipeline_trace.npz", "runs": pipe}

    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(gold, f, indent=0, separators=(",", ":"))
    print("wrote", os.path.join(OUT, "golden.json"))


if __name__ == "__main__":
    main()
