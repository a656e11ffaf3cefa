// The drop-in C++ API on the device: sspd::Rsea, merge_rseas, snapshots and
// run_detection, exercised the way the reference's own suites exercise the
// reference (proj/tests/test_rsea.cpp, test_snapshot.cpp, test_pipeline.cpp,
// acceptance.cpp), plus -- with HAVE_REF -- differential runs against the
// compiled reference through its C shim (bit-identical grids, identical
// report lists and estimates).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <random>
#include <set>
#include <sstream>
#include <thread>

#include "check.hpp"
#include "sspd/pipeline.hpp"
#include "sspd/rsea.hpp"
#include "sspd/snapshot.hpp"
#include "sspd/split.hpp"
#include "sspd_cuda.h"
#ifdef HAVE_REF
#include "ref_abi.hpp"
#endif

using namespace sspd;

namespace {

const RhfgConfig kCfg{10, 5, 8, 0xfeedULL};  // desk geometry
constexpr uint32_t kEta = 256;
constexpr double kTheta = 128;
constexpr uint32_t kK = 30;

std::vector<uint32_t> host_columns(const Rsea& g, uint32_t cip) {
  std::vector<uint32_t> cols;
  for (uint32_t i = 0; i < g.cfg().r; ++i) cols.push_back(rhfg(g.seeds(), i, cip, g.cfg()));
  return cols;
}

void plant(Rsea& g, uint32_t cip, uint32_t count, std::mt19937_64& rng) {
  std::set<uint32_t> oips;
  while (oips.size() < count) oips.insert(static_cast<uint32_t>(rng()));
  for (uint32_t oip : oips) g.update(cip, oip);
}

std::set<uint32_t> cips_of(const DetectionReport& r) {
  std::set<uint32_t> s;
  for (const auto& d : r.hosts) s.insert(d.cip);
  return s;
}

Rsea random_grid(std::mt19937_64& rng) {
  Rsea g(kCfg, kEta);
  std::vector<IpPair> p(5000);
  for (auto& x : p) x = {static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng())};
  g.scan_batch(p, 1);
  g.advance_slot(1);
  for (auto& x : p) x = {static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng())};
  g.scan_batch(p, 1);
  return g;
}

}  // namespace

TEST_CASE("update touches the r estimators at H1(oip)") {
  Rsea g(kCfg, kEta);
  const uint32_t cip = 0xC0A80101, oip = 0x08080808;
  g.update(cip, oip);
  const uint32_t bucket = hash_opposite(g.seeds(), oip, kEta);
  const auto cols = host_columns(g, cip);
  std::size_t zeroed = 0;
  for (Recorder v : std::as_const(g).cells()) zeroed += v == 0;
  CHECK(zeroed <= kCfg.r);
  for (uint32_t row = 0; row < kCfg.r; ++row) CHECK(std::as_const(g).estimator(row, cols[row])[bucket] == 0);
  Rsea again = g;
  again.update(cip, oip);
  CHECK(again == g);
  const uint32_t oip2 = 0x01010101;
  g.update(cip, oip2);
  const uint32_t b2 = hash_opposite(g.seeds(), oip2, kEta);
  CHECK(b2 != bucket);
  for (uint32_t row = 0; row < kCfg.r; ++row) CHECK(std::as_const(g).estimator(row, cols[row])[b2] == 0);
}

TEST_CASE("scan_batch is worker-count, batch and permutation invariant") {
  std::mt19937_64 rng(21);
  std::vector<IpPair> pairs(100000);
  for (auto& p : pairs) p = {static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng())};
  Rsea serial(kCfg, kEta);
  for (const auto& p : pairs) serial.update(p.cip, p.oip);
  for (unsigned w : {1u, 2u, 8u}) {
    Rsea par(kCfg, kEta);
    par.scan_batch(pairs, w);
    CHECK(par == serial);
  }
  Rsea fresh(kCfg, kEta);
  fresh.scan_batch({}, 4);
  CHECK(fresh == Rsea(kCfg, kEta));
  std::shuffle(pairs.begin(), pairs.end(), rng);
  Rsea shuffled(kCfg, kEta);
  shuffled.scan_batch(pairs, 3);
  CHECK(shuffled == serial);
  CHECK_THROWS_AS(fresh.scan_batch(pairs, 0), std::invalid_argument);
}

TEST_CASE("scan_records (B200 extension) equals scan_batch of the records' pairs") {
  std::mt19937_64 rng(22);
  std::vector<TraceRecord> recs(1100003);
  std::vector<IpPair> pairs(recs.size());
  for (std::size_t i = 0; i < recs.size(); ++i) {
    recs[i] = {static_cast<uint32_t>(i), static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng() % 5000)};
    pairs[i] = {recs[i].cip, recs[i].oip};
  }
  Rsea a(kCfg, kEta), b(kCfg, kEta);
  a.scan_batch(pairs, 1);
  b.scan_records(recs);
  b.scan_records({});
  CHECK(a == b);
  b.scan_records(std::span<const TraceRecord>(recs).subspan(17, 1001));
  CHECK(a == b);  // repeats within the slot
}

TEST_CASE("advance_slot: saturated fresh grid, equals element-wise increment") {
  Rsea g(kCfg, kEta);
  g.advance_slot(4);
  CHECK(g == Rsea(kCfg, kEta));
  std::mt19937_64 rng(22);
  Rsea base(kCfg, kEta);
  plant(base, 0x0A000001, 200, rng);
  Rsea expect = base;
  for (Recorder& v : expect.cells())
    if (v < kNeverSeen) ++v;  // writes through the mutable span
  for (unsigned v : {1u, 3u, 7u}) {
    Rsea grid = base;
    grid.advance_slot(v);
    CHECK(grid == expect);
  }
  CHECK_THROWS_AS(g.advance_slot(0), std::invalid_argument);
}

TEST_CASE("hot_sets") {
  Rsea g(kCfg, kEta);
  for (const auto& hs : g.hot_sets(kK, kTheta)) CHECK(hs.cols.empty());
  std::mt19937_64 rng(23);
  const uint32_t cip = 0xC0A80101;
  plant(g, cip, 2 * 128, rng);
  const auto cols = host_columns(g, cip);
  const auto hot = g.hot_sets(kK, kTheta);
  for (uint32_t row = 0; row < kCfg.r; ++row) {
    CHECK(hot[row].row == row);
    CHECK(std::find(hot[row].cols.begin(), hot[row].cols.end(), cols[row]) != hot[row].cols.end());
    CHECK(std::is_sorted(hot[row].cols.begin(), hot[row].cols.end()));
  }
  const auto wider = g.hot_sets(kK + 1, kTheta);
  for (uint32_t row = 0; row < kCfg.r; ++row)
    for (uint32_t c : hot[row].cols)
      CHECK(std::find(wider[row].cols.begin(), wider[row].cols.end(), c) != wider[row].cols.end());
}

TEST_CASE("finalize_candidate") {
  std::mt19937_64 rng(24);
  Rsea g(kCfg, kEta);
  const uint32_t cip = 0x0A141E28;
  plant(g, cip, 256, rng);
  const auto cols = host_columns(g, cip);
  const auto d = g.finalize_candidate(cols, kK, kTheta);
  REQUIRE(d.has_value());
  CHECK(d->cip == cip);
  CHECK(d->estimate >= kTheta);
  CHECK_FALSE(g.finalize_candidate(host_columns(g, 0x01020304), kK, kTheta).has_value());
  uint32_t cip2 = cip + 1;
  while (rhfg(g.seeds(), 0, cip2, kCfg) == cols[0]) ++cip2;
  plant(g, cip2, 256, rng);
  const auto cols2 = host_columns(g, cip2);
  std::vector<uint32_t> franken(kCfg.r);
  franken[0] = cols2[0];
  for (uint32_t i = 1; i < kCfg.r; ++i) franken[i] = recover_block(cols[0], cols[i]) ^ cols2[0];
  const auto f = g.finalize_candidate(franken, kK, kTheta);
  if (f) CHECK(rhfg(g.seeds(), 0, f->cip, kCfg) == franken[0]);
}

TEST_CASE("reconstruction finds exactly the planted host; strategies agree") {
  std::mt19937_64 rng(25);
  Rsea g(kCfg, kEta);
  const uint32_t cip = 0xC0A80101;
  plant(g, cip, 256, rng);
  for (int i = 0; i < 50; ++i) plant(g, static_cast<uint32_t>(rng()), 5, rng);
  const auto rec = g.reconstruct_recursive(kK, kTheta);
  CHECK(cips_of(rec) == std::set<uint32_t>{cip});
  for (unsigned w : {1u, 4u}) CHECK(cips_of(g.reconstruct_leveled(kK, kTheta, w)) == cips_of(rec));
  std::mt19937_64 r2(26);
  for (int trial = 0; trial < 20; ++trial) {
    Rsea s(kCfg, kEta);
    const int hosts = 1 + static_cast<int>(r2() % 6);
    for (int h = 0; h < hosts; ++h) plant(s, static_cast<uint32_t>(r2()), static_cast<uint32_t>(64 + r2() % 512), r2);
    CHECK(cips_of(s.reconstruct_recursive(kK, kTheta)) == cips_of(s.reconstruct_leveled(kK, kTheta, 3)));
  }
}

TEST_CASE("candidate buffer cap aborts with a diagnostic") {
  std::mt19937_64 rng(27);
  Rsea g(kCfg, kEta);
  for (int h = 0; h < 30; ++h) plant(g, static_cast<uint32_t>(rng()), 256, rng);
  g.set_candidate_cap(4);
  try {
    g.reconstruct_leveled(kK, kTheta, 2);
    FAIL("expected CandidateOverflow");
  } catch (const CandidateOverflow& e) {
    CHECK(e.count > 4);
    CHECK(e.level >= 2);
    CHECK(std::string(e.what()).find("candidate buffer cap exceeded at level") == 0);
  }
}

TEST_CASE("snapshot format") {
  Rsea fresh(kCfg, kEta);
  std::ostringstream out;
  export_snapshot(fresh, SnapshotMeta{kCfg.seed, 10, 5, 8, kEta, 30, 128, 0, 0}, out);
  const std::string bytes = out.str();
  REQUIRE(bytes.size() == kSnapshotHeaderSize + snapshot_payload_size(kEta, 5, 10));
  CHECK(std::all_of(bytes.begin() + kSnapshotHeaderSize, bytes.end(), [](char c) { return c == char(0xff); }));
  CHECK(snapshot_payload_size(1u << 11, 5, 14) == 335544320u);
  std::mt19937_64 rng(109);
  Rsea g(kCfg, kEta);
  for (int i = 0; i < 20000; ++i) g.update(static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng()));
  g.advance_slot(1);
  SnapshotMeta meta{kCfg.seed, 10, 5, 8, kEta, 30, 128, 1, 2};
  std::ostringstream o2;
  export_snapshot(g, meta, o2);
  std::istringstream in(o2.str());
  const auto imp = import_snapshot(in);
  CHECK(imp.rsea == g);
  CHECK(imp.meta.slot == 1);
  CHECK(imp.meta.node_id == 2);
  std::istringstream empty("");
  CHECK_THROWS_WITH_SUBSTR(import_snapshot(empty), "truncated header");
  std::string badmagic = o2.str();
  badmagic[0] = 'X';
  std::istringstream bm(badmagic);
  CHECK_THROWS_WITH_SUBSTR(import_snapshot(bm), "bad magic");
  std::string badver = o2.str();
  badver[4] = 9;
  std::istringstream bv(badver);
  CHECK_THROWS_WITH_SUBSTR(import_snapshot(bv), "unsupported version 9");
  std::string trunc = o2.str();
  trunc.resize(trunc.size() - 10);
  std::istringstream tr(trunc);
  CHECK_THROWS_WITH_SUBSTR(import_snapshot(tr), "truncated payload");
}

TEST_CASE("merge_rseas") {
  std::mt19937_64 rng(33);
  const Rsea one = random_grid(rng);
  CHECK(merge_rseas({&one}, MergePolicy::kUnionMin) == one);
  CHECK(merge_rseas({&one}, MergePolicy::kPaperMax) == one);
  Rsea full(kCfg, kEta);
  std::vector<Rsea> nodes(4, Rsea(kCfg, kEta));
  for (int slot = 0; slot < 3; ++slot) {
    for (int i = 0; i < 4000; ++i) {
      const uint32_t c = static_cast<uint32_t>(rng()), o = static_cast<uint32_t>(rng());
      full.update(c, o);
      nodes[rng() % 4].update(c, o);
    }
    full.advance_slot(1);
    for (auto& n : nodes) n.advance_slot(1);
  }
  const Rsea merged = merge_rseas({&nodes[0], &nodes[1], &nodes[2], &nodes[3]}, MergePolicy::kUnionMin);
  CHECK(merged == full);
  const Rsea mx = merge_rseas({&nodes[0], &nodes[1], &nodes[2], &nodes[3]}, MergePolicy::kPaperMax);
  CHECK_FALSE(mx == full);
  const Rsea a = random_grid(rng), b = random_grid(rng), c = random_grid(rng);
  const Rsea ab = merge_rseas({&a, &b}, MergePolicy::kUnionMin);
  CHECK(ab == merge_rseas({&b, &a}, MergePolicy::kUnionMin));
  const Rsea bc = merge_rseas({&b, &c}, MergePolicy::kUnionMin);
  CHECK(merge_rseas({&ab, &c}, MergePolicy::kUnionMin) == merge_rseas({&a, &bc}, MergePolicy::kUnionMin));
  CHECK(merge_rseas({&a, &a}, MergePolicy::kUnionMin) == a);
  Rsea other(RhfgConfig{10, 5, 8, 0xdefULL}, kEta);
  CHECK_THROWS_AS(merge_rseas({&a, &other}, MergePolicy::kUnionMin), std::invalid_argument);
  CHECK_THROWS_AS(merge_rseas({}, MergePolicy::kUnionMin), std::invalid_argument);
}

namespace {

RunConfig test_config() {
  RunConfig rc = desk_preset();
  rc.cfg.seed = 0x5eedULL;
  rc.window.k = 5;
  rc.alpha = 1024;
  return rc;
}

SynthResult workload(uint32_t supers, uint32_t count, uint32_t slots, const RunConfig& rc, uint64_t seed) {
  SynthSpec spec;
  spec.slots = slots;
  for (uint32_t i = 0; i < supers; ++i) spec.planted.push_back({0x0A000000 + i, count, 0, slots - 1});
  spec.background_hosts = 200;
  spec.pairs_per_slot = 500;
  spec.max_distinct_per_host = 8;
  return synth_trace(spec, seed, rc.window);
}

std::vector<std::vector<TraceRecord>> split(const std::vector<TraceRecord>& t, unsigned n, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<std::vector<TraceRecord>> s(n);
  for (const auto& r : t) s[rng() % n].push_back(r);
  return s;
}

}  // namespace

TEST_CASE("pipeline: empty, invalid, planted supers in every window") {
  CHECK(run_detection({{}}, test_config()).empty());
  RunConfig bad = test_config();
  bad.cfg.q = 8;
  CHECK_THROWS_AS(run_detection({{}}, bad), std::invalid_argument);
  CHECK_THROWS_AS(run_detection({}, test_config()), std::invalid_argument);
  const RunConfig rc = test_config();
  const auto w = workload(3, 256, 8, rc, 77);
  const auto reps = run_detection({w.trace}, rc);
  REQUIRE(reps.size() == 8);
  for (const auto& r : reps)
    for (uint32_t i = 0; i < 3; ++i) CHECK(cips_of(r).count(0x0A000000 + i) == 1);
}

TEST_CASE("pipeline: strategies and worker counts agree") {
  RunConfig rc = test_config();
  const auto w = workload(2, 256, 5, rc, 78);
  rc.strategy = Strategy::kRecursive;
  const auto a = run_detection({w.trace}, rc);
  rc.strategy = Strategy::kLeveled;
  rc.workers = 4;
  const auto b = run_detection({w.trace}, rc);
  REQUIRE(a.size() == b.size());
  for (std::size_t s = 0; s < a.size(); ++s) {
    CHECK(cips_of(a[s]) == cips_of(b[s]));
    REQUIRE(a[s].hosts.size() == b[s].hosts.size());
    for (std::size_t h = 0; h < a[s].hosts.size(); ++h) CHECK(a[s].hosts[h].estimate == b[s].hosts[h].estimate);
  }
}

TEST_CASE("union-min over several routers (B200 extension): same reports as one grid") {
  RunConfig rc = test_config();
  const auto w = workload(3, 256, 10, rc, 91);
  const auto shards = split(w.trace, 4, 92);
  const auto one = run_detection(shards, rc);
  const auto single_trace = run_detection({w.trace}, rc);
  for (const char* routers : {"2", "3", "4"}) {
    setenv("SSPD_ROUTERS", routers, 1);  // several routers on this one device
    const auto many = run_detection(shards, rc);
    const auto split_trace = run_detection({w.trace}, rc);
    unsetenv("SSPD_ROUTERS");
    REQUIRE(many.size() == one.size());
    REQUIRE(split_trace.size() == single_trace.size());
    for (std::size_t s = 0; s < one.size(); ++s) {
      REQUIRE(many[s].hosts.size() == one[s].hosts.size());
      CHECK(many[s].slot == one[s].slot);
      for (std::size_t h = 0; h < one[s].hosts.size(); ++h) {
        CHECK(many[s].hosts[h].cip == one[s].hosts[h].cip);
        CHECK(many[s].hosts[h].estimate == one[s].hosts[h].estimate);
      }
      REQUIRE(split_trace[s].hosts.size() == single_trace[s].hosts.size());
      for (std::size_t h = 0; h < single_trace[s].hosts.size(); ++h)
        CHECK(split_trace[s].hosts[h].estimate == single_trace[s].hosts[h].estimate);
    }
  }
}

TEST_CASE("narrow stamps (B200 extension): same reports, distances refused") {
  RunConfig rc = test_config();
  const auto w = workload(3, 256, 12, rc, 79);
  const auto wide = run_detection({w.trace}, rc);
  for (uint32_t bits : {8u, 16u}) {
    rc.stamp_bits = bits;
    const auto narrow = run_detection(split(w.trace, 3, 82), rc);
    REQUIRE(narrow.size() == wide.size());
    for (std::size_t s = 0; s < wide.size(); ++s) {
      REQUIRE(narrow[s].hosts.size() == wide[s].hosts.size());
      for (std::size_t h = 0; h < wide[s].hosts.size(); ++h) {
        CHECK(narrow[s].hosts[h].cip == wide[s].hosts[h].cip);
        CHECK(narrow[s].hosts[h].estimate == wide[s].hosts[h].estimate);
      }
    }
    rc.policy = MergePolicy::kPaperMax;  // needs full stamps for merge_rseas
    CHECK_THROWS_AS(run_detection(split(w.trace, 2, 83), rc), std::invalid_argument);
    rc.policy = MergePolicy::kUnionMin;
  }
  Rsea g(kCfg, kEta, StampWidth{8, kK});
  CHECK(g.stamp_width().bits == 8);
  CHECK(g.stamp_width().window == kK);
  std::mt19937_64 rng(5);
  plant(g, 0x0A0B0C0D, 300, rng);
  CHECK(cips_of(g.reconstruct_leveled(kK, kTheta, 1)).count(0x0A0B0C0D) == 1);
  CHECK_THROWS_AS(g.cells(), std::invalid_argument);
  CHECK_THROWS_AS(Rsea{g}, std::invalid_argument);
  CHECK_THROWS_AS((Rsea(kCfg, kEta, StampWidth{8, 0})), std::invalid_argument);
  CHECK_THROWS_AS((Rsea(kCfg, kEta, StampWidth{12, 5})), std::invalid_argument);
}

TEST_CASE("pipeline: 4-way union-min sharding equals the single-node run") {
  const RunConfig rc = test_config();
  const auto w = workload(3, 256, 6, rc, 80);
  const auto shards = split(w.trace, 4, 81);
  std::vector<std::vector<Recorder>> g1, g4;
  const auto single = run_detection({w.trace}, rc, [&](uint64_t, const Rsea& g) {
    g1.emplace_back(g.cells().begin(), g.cells().end());
  });
  const auto multi = run_detection(shards, rc, [&](uint64_t, const Rsea& g) {
    g4.emplace_back(g.cells().begin(), g.cells().end());
  });
  REQUIRE(single.size() == multi.size());
  REQUIRE(g1.size() == g4.size());
  for (std::size_t s = 0; s < single.size(); ++s) {
    CHECK(g1[s] == g4[s]);
    CHECK(cips_of(single[s]) == cips_of(multi[s]));
  }
}

TEST_CASE("pipeline: split super point detected only globally") {
  RunConfig rc = test_config();
  const uint32_t cip = 0xC0A80101;
  std::vector<std::vector<TraceRecord>> shards(4);
  for (uint32_t i = 0; i < 256; ++i) shards[i % 4].push_back({0, cip, 0x40000000 + i});
  for (const auto& s : shards) {
    const auto solo = run_detection({s}, rc);
    REQUIRE(solo.size() == 1);
    CHECK(cips_of(solo[0]).count(cip) == 0);
  }
  const auto global = run_detection(shards, rc);
  REQUIRE(global.size() == 1);
  CHECK(cips_of(global[0]).count(cip) == 1);
  rc.policy = MergePolicy::kPaperMax;  // the intersection loses it
  CHECK(cips_of(run_detection(shards, rc)[0]).count(cip) == 0);
}

TEST_CASE("concurrent SCAN-phase callers (rsea.hpp:49-51) give the serial grid") {
  std::mt19937_64 rng(90);
  std::vector<IpPair> pairs(200000);
  for (auto& p : pairs) p = {static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng())};
  Rsea serial(kCfg, kEta);
  serial.scan_batch(pairs, 1);
  Rsea shared(kCfg, kEta);
  std::vector<std::thread> th;
  for (int t = 0; t < 8; ++t)
    th.emplace_back([&, t] {
      const std::size_t lo = pairs.size() * t / 8, hi = pairs.size() * (t + 1) / 8;
      if (t % 2)  // half the threads batch, half update one by one
        shared.scan_batch(std::span<const IpPair>(pairs.data() + lo, hi - lo), 2);
      else
        for (std::size_t i = lo; i < hi; ++i) shared.update(pairs[i].cip, pairs[i].oip);
    });
  for (auto& x : th) x.join();
  CHECK(shared == serial);
}

TEST_CASE("concurrent scans into separate grids share the host packing pool") {
  // pageable batches >= 4096 pairs are packed into pinned staging by one
  // process-wide worker pool; four threads scanning four grids at once (pairs
  // and records, several chunks each) must each get its serial grid
  std::mt19937_64 rng(95);
  std::vector<TraceRecord> recs(700001);
  for (auto& r : recs) r = {0, static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng() % 100000)};
  std::vector<IpPair> pairs(recs.size());
  for (std::size_t i = 0; i < recs.size(); ++i) pairs[i] = {recs[i].cip, recs[i].oip};
  Rsea serial(kCfg, kEta);
  serial.scan_batch(pairs, 1);
  std::vector<Rsea> grids;
  for (int t = 0; t < 4; ++t) grids.emplace_back(kCfg, kEta);
  std::vector<std::thread> th;
  for (int t = 0; t < 4; ++t)
    th.emplace_back([&, t] {
      for (int rep = 0; rep < 3; ++rep) {
        if (t % 2)
          grids[t].scan_records(recs);
        else
          grids[t].scan_batch(pairs, 1);
      }
    });
  for (auto& x : th) x.join();
  for (const Rsea& g : grids) CHECK(g == serial);
}

TEST_CASE("Rsea value semantics: copies are independent, moves keep the state") {
  std::mt19937_64 rng(91);
  Rsea a(kCfg, kEta);
  plant(a, 0x0A0B0C0D, 300, rng);
  Rsea b = a;            // copy
  b.advance_slot(1);
  CHECK_FALSE(a == b);
  Rsea c = std::move(b); // move keeps b's state
  Rsea d(kCfg, kEta);
  d = a;                 // copy-assign
  d.advance_slot(1);
  CHECK(c == d);
  d = std::move(c);      // move-assign
  CHECK(d.reconstruct_leveled(kK, kTheta, 1).hosts.size() == a.reconstruct_leveled(kK, kTheta, 1).hosts.size());
  // writes through a mutable span are seen by the device, later updates too
  auto cells = a.cells();
  std::fill(cells.begin(), cells.end(), kNeverSeen);
  a.update(1, 2);
  std::size_t zeros = 0;
  for (Recorder v : std::as_const(a).cells()) zeros += v == 0;
  CHECK(zeros >= 1);
  CHECK(zeros <= kCfg.r);
}

#ifdef HAVE_REF
namespace {

struct RefRows {
  std::vector<uint64_t> slots;
  std::vector<uint32_t> cips;
  std::vector<double> ests;
  size_t n_reports = 0;
};

RefRows ref_pipeline(const std::vector<std::vector<TraceRecord>>& shards, const RunConfig& rc) {
  std::vector<uint32_t> recs;
  std::vector<size_t> off{0};
  for (const auto& s : shards) {
    for (const auto& r : s) recs.insert(recs.end(), {r.ts, r.cip, r.oip});
    off.push_back(recs.size() / 3);
  }
  RefRows out;
  const size_t cap = 1 << 20;
  out.slots.resize(cap);
  out.cips.resize(cap);
  out.ests.resize(cap);
  size_t n = 0;
  const int rcode = ref_run_detection(rc.cfg.q, rc.cfg.r, rc.cfg.delta, rc.cfg.seed, rc.eta, rc.window.mu,
                                      rc.window.k, rc.window.start, rc.theta, rc.alpha, 1,
                                      rc.policy == MergePolicy::kUnionMin ? 0 : 1,
                                      rc.strategy == Strategy::kLeveled ? 1 : 0, rc.candidate_cap, recs.data(),
                                      off.data(), shards.size(), out.slots.data(), out.cips.data(),
                                      out.ests.data(), cap, &n, &out.n_reports);
  if (rcode != 0) throw std::runtime_error(std::string("reference failed: ") + ref_last_error());
  out.slots.resize(n);
  out.cips.resize(n);
  out.ests.resize(n);
  return out;
}

void expect_same(const std::vector<DetectionReport>& ours, const RefRows& ref) {
  REQUIRE(ours.size() == ref.n_reports);
  size_t i = 0;
  for (const auto& rep : ours)
    for (const auto& h : rep.hosts) {
      REQUIRE(i < ref.cips.size());
      CHECK(ref.slots[i] == rep.slot);
      CHECK(ref.cips[i] == h.cip);
      CHECK(ref.ests[i] == h.estimate);  // bit-identical doubles
      ++i;
    }
  CHECK(i == ref.cips.size());
}

}  // namespace

TEST_CASE("differential: grids bit-identical to the compiled reference") {
  for (const RhfgConfig& cfg : {RhfgConfig{10, 5, 8, 0x5eed}, RhfgConfig{14, 5, 6, 0x5eed}, RhfgConfig{12, 7, 4, 3}}) {
    const uint32_t eta = cfg.q == 12 ? 1000 : (cfg.q == 10 ? 256 : 2048);
    Rsea g(cfg, eta);
    void* r = ref_grid_create(cfg.q, cfg.r, cfg.delta, cfg.seed, eta);
    std::mt19937_64 rng(7);
    std::vector<uint16_t> want(ref_grid_size(r));
    for (int step = 0; step < 3; ++step) {
      std::vector<IpPair> p(60000);
      for (auto& x : p) x = {static_cast<uint32_t>(rng()), static_cast<uint32_t>(rng())};
      g.scan_batch(p, 1);
      ref_scan(r, reinterpret_cast<const uint32_t*>(p.data()), p.size(), 4);
      ref_get_cells(r, want.data());
      const auto got = std::as_const(g).cells();
      CHECK(std::equal(got.begin(), got.end(), want.begin()));
      g.advance_slot(1);
      ref_advance(r, 4);
    }
    ref_grid_destroy(r);
  }
}

TEST_CASE("differential: run_detection reports equal the reference (single, 4 shards, paper-max)") {
  const RunConfig rc = test_config();
  const auto w = workload(3, 256, 8, rc, 77);
  expect_same(run_detection({w.trace}, rc), ref_pipeline({w.trace}, rc));
  const auto shards = split(w.trace, 4, 81);
  expect_same(run_detection(shards, rc), ref_pipeline(shards, rc));
  RunConfig pm = rc;
  pm.policy = MergePolicy::kPaperMax;
  expect_same(run_detection(shards, pm), ref_pipeline(shards, pm));
  RunConfig rec = rc;
  rec.strategy = Strategy::kRecursive;
  expect_same(run_detection({w.trace}, rec), ref_pipeline({w.trace}, rec));
  // shards that are not time sorted (the record-by-record walk; sorted shards
  // take a binary search per slot) and a trace with empty slots
  auto unsorted = shards;
  std::mt19937_64 rng(83);
  for (int i = 0; i < 40; ++i) {
    auto& s = unsorted[rng() % unsorted.size()];
    std::swap(s[rng() % s.size()], s[rng() % s.size()]);
  }
  expect_same(run_detection(unsorted, rc), ref_pipeline(unsorted, rc));
  expect_same(run_detection(unsorted, pm), ref_pipeline(unsorted, pm));
  std::vector<TraceRecord> gappy;
  for (const TraceRecord& r : w.trace)
    if (r.ts % 3 != 1) gappy.push_back({r.ts * 2, r.cip, r.oip});
  expect_same(run_detection({gappy}, rc), ref_pipeline({gappy}, rc));
  expect_same(run_detection(split(gappy, 3, 85), rc), ref_pipeline(split(gappy, 3, 85), rc));
}

TEST_CASE("differential: acceptance end-to-end at the paper's parameters") {
  // acceptance.cpp:123-167 (criterion 4): 35 slots, 20 supers at 2*theta,
  // 50k Zipf background hosts; recall 1.0 and mean FPR <= 0.05, and every
  // report identical to the reference's.
  RunConfig rc;
  rc.cfg = RhfgConfig{14, 5, 6, 0x60D5EEDULL};
  rc.eta = 1u << 11;
  rc.theta = 1024;
  rc.window.k = 30;
  SynthSpec spec;
  spec.slots = 35;
  for (uint32_t i = 0; i < 20; ++i) spec.planted.push_back({0x0A000000 + i * 1000, 2048, 0, 34});
  spec.background_hosts = 50000;
  spec.zipf_exponent = 1.1;
  spec.pairs_per_slot = 20000;
  spec.max_distinct_per_host = 64;
  const auto w = synth_trace(spec, 104, rc.window);
  const auto reps = run_detection({w.trace}, rc);
  REQUIRE(reps.size() == 35);
  double fpr = 0;
  for (const auto& r : reps) {
    std::unordered_set<uint32_t> rep;
    for (const auto& d : r.hosts) rep.insert(d.cip);
    for (const auto& p : spec.planted) CHECK(rep.count(p.cip) == 1);
    fpr += evaluate(rep, w.truth.slots[r.slot], rc.theta).fpr;
  }
  CHECK(fpr / reps.size() <= 0.05);
  expect_same(reps, ref_pipeline({w.trace}, rc));
}

// Config C1 at its stated size (bench.py --config c1): 10 slots x
// 1e6 pairs (uniform, with 20 planted supers x 2048 distinct oips first),
// the reference defaults q14 r5 delta6 eta2048, k=5, theta=1024.  Through
// sspd::run_detection against the compiled reference (pipeline.cpp:16-89):
// every slot's full grid (167,772,160 recorders), all 81,920 R_k and every
// report; then the probe-less (pipelined) run against ref_run_detection.
TEST_CASE("differential: C1 at full size, every slot's grid, R_k and reports") {
  RunConfig rc;
  rc.cfg = RhfgConfig{14, 5, 6, 0x5eed};
  rc.eta = 2048;
  rc.window.k = 5;
  rc.theta = 1024;
  constexpr uint32_t kSlots = 10;
  constexpr uint64_t kPairs = 1'000'000;
  sspd_synth_params_t sp{0x5eedULL ^ 0xC2C2, 1, 0, 20, 2048, kPairs, 0, 1};
  std::vector<uint64_t> cdf(1);
  REQUIRE(sspd_synth_zipf_cdf(1, 1.1, cdf.data()) == SSPD_OK);
  std::vector<TraceRecord> trace;
  trace.reserve(kSlots * kPairs);
  std::vector<std::vector<uint32_t>> slot_pairs(kSlots, std::vector<uint32_t>(2 * kPairs));
  for (uint32_t s = 0; s < kSlots; ++s) {
    REQUIRE(sspd_synth_host(&sp, cdf.data(), s, 0, kPairs, slot_pairs[s].data()) == SSPD_OK);
    for (uint64_t j = 0; j < kPairs; ++j) trace.push_back({s, slot_pairs[s][2 * j], slot_pairs[s][2 * j + 1]});
  }
  const unsigned workers = std::max(1u, std::thread::hardware_concurrency());
  void* ref = ref_grid_create(14, 5, 6, 0x5eed, 2048);
  const size_t n_rec = ref_grid_size(ref);
  REQUIRE(n_rec == 167772160u);
  std::vector<uint16_t> want(n_rec);
  const size_t n_cells = size_t{5} << 14;
  std::vector<uint32_t> rk(n_cells);
  uint64_t probed = 0, cells_ok = 0, rk_ok = 0;
  const auto reps = run_detection({trace}, rc, [&](uint64_t slot, const Rsea& grid) {
    ref_scan(ref, slot_pairs[slot].data(), kPairs, workers);
    ref_get_cells(ref, want.data());
    const auto got = grid.cells();
    cells_ok += got.size() == want.size() && std::equal(got.begin(), got.end(), want.begin());
    REQUIRE(sspd_active_counts(grid.handle(), rc.window.k, rk.data()) == SSPD_OK);
    bool same = true;
    for (size_t c = 0; c < n_cells && same; ++c) {
      uint32_t n = 0;
      for (size_t b = 0; b < rc.eta; ++b) n += want[c * rc.eta + b] < rc.window.k;
      same = n == rk[c];
    }
    rk_ok += same;
    ++probed;
    ref_advance(ref, workers);
  });
  ref_grid_destroy(ref);
  CHECK(probed == kSlots);
  CHECK(cells_ok == kSlots);
  CHECK(rk_ok == kSlots);
  const RefRows want_reps = ref_pipeline({trace}, rc);
  expect_same(reps, want_reps);
  expect_same(run_detection({trace}, rc), want_reps);  // no probe: the pipelined path
  size_t hosts = 0;
  for (const auto& r : reps) hosts += r.hosts.size();
  std::cerr << "  C1: " << kSlots << " slots x " << kPairs << " pairs, " << hosts
            << " reports, grids / R_k / reports identical every slot\n";
  CHECK(hosts >= 20 * kSlots);
}

// A window the ring cannot budget (K > eta/4): run_detection
// tracks no ring and counts over the stamps instead -- the reference's
// largest legal k at its default geometry, whose ring would need
// 4 B x 65534 x 5 x 2^14 = 21 GB.  Reports equal the reference's.
TEST_CASE("differential: run_detection at k = 65534 without a window ring") {
  RunConfig rc;
  rc.cfg = RhfgConfig{14, 5, 6, 0x5eed};
  rc.eta = 2048;
  rc.theta = 1024;
  rc.window.k = 65534;
  const auto w = workload(3, 1500, 4, rc, 123);
  expect_same(run_detection({w.trace}, rc), ref_pipeline({w.trace}, rc));
  RunConfig desk = test_config();
  desk.window.k = 65534;
  const auto wd = workload(3, 256, 6, desk, 124);
  expect_same(run_detection({wd.trace}, desk), ref_pipeline({wd.trace}, desk));
  const auto shards = split(wd.trace, 3, 125);
  expect_same(run_detection(shards, desk), ref_pipeline(shards, desk));
}

// export_snapshot byte for byte against the reference's (snapshot.cpp:36-68):
// the same scans and advances into our device grid and the compiled
// reference's grid, the same meta -> identical 56-byte header and u16 payload;
// and each import of the other's bytes reproduces the grid.
TEST_CASE("differential: export_snapshot bytes equal the reference's") {
  for (const RhfgConfig& cfg : {RhfgConfig{10, 5, 8, 0x5eed}, RhfgConfig{14, 5, 6, 0xabc}}) {
    const uint32_t eta = cfg.q == 10 ? 256 : 2048;
    Rsea g(cfg, eta);
    void* r = ref_grid_create(cfg.q, cfg.r, cfg.delta, cfg.seed, eta);
    std::mt19937_64 rng(cfg.seed);
    for (int step = 0; step < 4; ++step) {
      std::vector<IpPair> p(40000);
      for (auto& x : p) x = {static_cast<uint32_t>(rng() % 5000), static_cast<uint32_t>(rng())};
      g.scan_batch(p, 1);
      ref_scan(r, reinterpret_cast<const uint32_t*>(p.data()), p.size(), 4);
      if (step < 3) {
        g.advance_slot(1);
        ref_advance(r, 4);
      }
    }
    SnapshotMeta m;
    m.k = 5;
    m.theta = 128;
    m.slot = 3;
    m.node_id = 7;
    std::ostringstream ours(std::ios::out | std::ios::binary);
    export_snapshot(g, m, ours);
    const std::string a = ours.str();
    std::string b(a.size() + 64, '\0');
    const size_t n = ref_export_snapshot(r, 5, 128, 3, 7, b.data(), b.size());
    REQUIRE(n == a.size());
    b.resize(n);
    CHECK(a.size() == kSnapshotHeaderSize + snapshot_payload_size(eta, cfg.r, cfg.q));
    CHECK(a == b);
    std::istringstream back(b, std::ios::in | std::ios::binary);
    const ImportedSnapshot imp = import_snapshot(back);
    CHECK(imp.rsea == g);
    CHECK(imp.meta.node_id == 7u);
    ref_grid_destroy(r);
  }
}
#endif

CHECK_MAIN
