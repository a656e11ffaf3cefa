"""The CPU oracle (oracle/sspd_oracle.c) pinned against the golden vectors
generated from the compiled reference (tests/golden/make_golden.py), and --
where oracle/_ref was built -- against the reference directly.  No GPU."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD_DIR = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD_DIR, "golden.json")) as f:
        return json.load(f)


def test_survey_anchors():
    """Hand anchors recorded in SURVEY.md §8c from the reference."""
    assert O.h1_raw(0x5eed, 0x08080808) == 0x48d9a5b7829ca305
    assert O.row0_raw(0x5eed, 0xC0A80101) == 0x3a77151ffcf0dfdb
    assert O.rhfg_cols(14, 5, 6, 0x5eed, 0xC0A80101) == [8155, 7898, 16351, 5467, 12273]
    assert O.rhfg_cols(10, 5, 8, 0x5eed, 0xC0A80101) == [987, 730, 986, 883, 795]
    assert O.hot_cutoff(2048, 1024) == 806
    assert O.hot_cutoff(256, 128) == 101
    assert O.estimate_cardinality(2048, 806) == 1024.2882020679153
    assert O.blocks_consistent(14, 5, 6, 0x3f00, 0x0001) is False


def test_hashes(gold):
    ks = gold["keys"]
    for seed_hex, tabs in gold["hash"].items():
        seed = int(seed_hex, 16)
        assert [hex(O.h1_raw(seed, k)) for k in ks] == tabs["h1"]
        assert [hex(O.row0_raw(seed, k)) for k in ks] == tabs["row0"]


def test_hash_opposite(gold):
    ks = gold["keys"]
    L = O.lib()
    for key, vals in gold["hash_opposite"].items():
        seed_hex, eta = key.split(":")
        s = O._CSeeds()
        L.so_seeds_init(O.C.byref(s), O.C.c_uint64(int(seed_hex, 16)))
        got = [L.so_hash_opposite(O.C.byref(s), O.C.c_uint32(k), O.C.c_uint32(int(eta)))
               for k in ks]
        assert got == vals, key


def test_rhfg(gold):
    ks = gold["keys"]
    for key, rows in gold["rhfg"].items():
        q, r, d, s = key.split(",")
        q, r, d, s = int(q), int(r), int(d), int(s, 16)
        assert [O.rhfg_cols(q, r, d, s, k) for k in ks] == rows, key


def test_assemble_and_blocks(gold):
    for q, r, d, blocks, ip in gold["assemble"]:
        assert O.assemble_ip(q, r, d, blocks) == ip, (q, r, d, blocks)
    for q, r, d, lo, hi, want in gold["blocks_consistent"]:
        assert O.blocks_consistent(q, r, d, lo, hi) == bool(want)


def test_cutoff_estimate_validate(gold):
    for eta, th, want in gold["hot_cutoff"]:
        assert O.hot_cutoff(eta, th) == want
    for eta, rk, want in gold["estimate"]:
        assert O.estimate_cardinality(eta, rk).hex() == want
    for args, n, msg in gold["validate"]:
        q, r, d, eta, k, th = args
        got_n, got_msg = O.validate_config(q, r, d, eta, k, th)
        assert (got_n, got_msg) == (n, msg), args


def test_grid_sequences(gold):
    for case in gold["grids"]:
        q, r, d, eta, seed = case["cfg"]
        g = O.OracleGrid(q, r, d, int(seed, 16), eta)
        rng = O.Mt64(case["mt_seed"])
        for step in case["steps"]:
            g.scan(rng.pairs(case["pairs_per_step"]))
            c = g.cells()
            assert hex(O.fnv1a64(c)) == step["fnv"], case["name"]
            assert int((c == 0).sum()) == step["zeros"]
            g.advance()


def test_planted_states(gold):
    rng = O.Mt64(gold["states"]["mt_seed"])
    for st, case in enumerate(gold["states"]["list"]):
        q, r, d, eta, seed = case["cfg"]
        g = O.OracleGrid(q, r, d, int(seed, 16), eta)
        hosts = int(rng.next() % 8)
        for _ in range(hosts):
            cip = int(rng.next()) & 0xFFFFFFFF
            cnt = 32 + int(rng.next() % 512)
            g.scan(np.stack([np.full(cnt, cip, np.uint32), rng.draw(cnt).astype(np.uint32)], 1))
        g.scan(rng.pairs(2000))
        if st % 3 == 0:
            g.advance()
        assert hex(O.fnv1a64(g.cells())) == case["cells_fnv"]
        for k, want in case["counts_fnv"].items():
            assert hex(O.fnv1a64(g.active_counts(int(k)))) == want
        assert [h.tolist() for h in g.hot_sets(30, 128.0)] == case["hot"]
        lev = [[x.cip, x.estimate.hex()] for x in g.reconstruct(30, 128.0)]
        rec = [[x.cip, x.estimate.hex()] for x in g.reconstruct(30, 128.0, leveled=False)]
        assert lev == case["leveled"]
        assert rec == case["recursive"]


def test_overflow(gold):
    ov = gold["overflow"]
    g = O.OracleGrid(10, 5, 8, 0xfeed, 256)
    rng = O.Mt64(ov["mt_seed"])
    for _ in range(ov["hosts"]):
        cip = int(rng.next()) & 0xFFFFFFFF
        g.scan(np.stack([np.full(ov["count"], cip, np.uint32),
                         rng.draw(ov["count"]).astype(np.uint32)], 1))
    for cap, want in ov["caps"].items():
        if want is None:
            g.reconstruct(30, 128.0, cap=int(cap))
        else:
            with pytest.raises(O.CandidateOverflow) as e:
                g.reconstruct(30, 128.0, cap=int(cap))
            assert [e.value.level, e.value.count] == want


def test_pipeline(gold):
    p = gold["pipeline"]
    z = np.load(os.path.join(GOLD_DIR, p["trace"]))
    trace, owner = z["trace"], z["owner"]
    shards = [trace[owner == i] for i in range(4)]
    for label, recs, pol in [("single", [trace], 0), ("sharded_union", shards, 0),
                             ("sharded_paper", shards, 1)]:
        n_slots, rows = O.run_detection(recs, q=10, r=5, delta=8, seed=0x5eed, eta=256, mu=1.0,
                                        k=5, theta=128.0, policy=pol)
        want = p["runs"][label]
        assert n_slots == want["n_reports"]
        assert [[s, d.cip, d.estimate.hex()] for s, d in rows] == want["rows"], label


def test_merge_algebra():
    """test_snapshot.cpp:132-144 on the oracle."""
    rng = O.Mt64(33)
    grids = []
    for _ in range(3):
        g = O.OracleGrid(10, 5, 8, 0xfeed, 256)
        g.scan(rng.pairs(3000))
        g.advance()
        g.scan(rng.pairs(3000))
        grids.append(g)
    a, b, c = grids
    ab = O.OracleGrid.merge([a, b])
    assert ab == O.OracleGrid.merge([b, a])
    assert O.OracleGrid.merge([ab, c]) == O.OracleGrid.merge([a, O.OracleGrid.merge([b, c])])
    assert O.OracleGrid.merge([a, a]) == a
    with pytest.raises(ValueError):
        O.OracleGrid.merge([a, O.OracleGrid(10, 5, 8, 0xdef, 256)])


def test_mt64_matches_std():
    # first outputs of std::mt19937_64 with the default seed 5489
    m = O.Mt64(5489)
    assert m.next() == 14514284786278117030


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_compiled_reference_random():
    """Direct differential run: random geometry, seeds and traffic."""
    rng = np.random.default_rng(1234)
    for trial in range(6):
        q = int(rng.integers(9, 15))
        d = int(rng.integers(2, q))
        r = max(3, -(-(32 - q) // d) + 2)
        eta = int(rng.choice([64, 100, 256, 333]))
        seed = int(rng.integers(0, 2**63))
        o = O.OracleGrid(q, r, d, seed, eta)
        f = O.RefGrid(q, r, d, seed, eta)
        mt = O.Mt64(trial)
        for s in range(3):
            for h in range(3):
                cip = int(mt.next()) & 0xFFFFFFFF
                pr = np.stack([np.full(200, cip, np.uint32), mt.draw(200).astype(np.uint32)], 1)
                o.scan(pr)
                f.scan(pr, workers=3)
            p = mt.pairs(5000)
            o.scan(p)
            f.scan(p, workers=2)
            assert np.array_equal(o.cells(), f.cells())
            for k in (1, 2, 3):
                th = float(eta) / 3
                assert [x.tolist() for x in o.hot_sets(k, th)] == \
                    [x.tolist() for x in f.hot_sets(k, th)]
                a = [(x.cip, x.estimate) for x in o.reconstruct(k, th)]
                b = [(x.cip, x.estimate) for x in f.reconstruct(k, th, workers=2)]
                assert a == b
            o.advance()
            f.advance(2)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_python_validate_config_equals_reference():
    """The Python host mirror's validate_config (paper_1803_11036_b200/pipeline.py)
    returns the compiled reference's full message list (hashing.cpp:63-87) on the
    same 120,384-point grid the C++ differential uses (tests/cpp/test_api_host.cpp)."""
    from paper_1803_11036_b200.pipeline import validate_config

    n = 0
    for q in range(19):
        for r in range(9):
            for d in range(q + 2):
                for eta in (0, 1, 2, 256):
                    for k in (0, 1, 65534, 65535):
                        for th in (0.0, 0.5, 1.0, 1024.0):
                            assert validate_config(q, r, d, eta, k, th) == \
                                O.ref_validate_all(q, r, d, eta, k, th), (q, r, d, eta, k, th)
                            n += 1
    assert n == 120384
