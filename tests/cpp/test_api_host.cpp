// Host-only parts of the drop-in C++ API (no GPU needed): hashing, estimator
// helpers, the work split and the workload utilities.  Cases follow the
// reference suites (proj/tests/test_hashing.cpp, test_estimator.cpp,
// test_workload.cpp, acceptance.cpp:353-383); with HAVE_REF the synthetic
// generator is also checked record-for-record against the compiled reference.
#include <cmath>
#include <cstring>
#include <iostream>
#include <random>
#include <set>
#include <sstream>

#include "check.hpp"
#include "sspd/estimator.hpp"
#include "sspd/hashing.hpp"
#include "sspd/split.hpp"
#include "sspd/workload.hpp"
#ifdef HAVE_REF
#include "ref_abi.hpp"
#endif

using namespace sspd;

namespace {
const RhfgConfig kPaper{14, 5, 6, 0x1234abcdULL};
const RhfgConfig kDesk{10, 5, 8, 0x1234abcdULL};
uint32_t slice(uint32_t cip, uint32_t i, const RhfgConfig& c) {
  return (cip >> ((i - 1) * c.delta)) & c.column_mask();
}
}  // namespace

TEST_CASE("survey anchors of the reference hashing") {
  HashSeeds s(0x5eed);
  CHECK(s.h1_raw(0x08080808) == 0x48d9a5b7829ca305ULL);
  CHECK(s.row0_raw(0xC0A80101) == 0x3a77151ffcf0dfdbULL);
  CHECK(hash_opposite(s, 0x08080808, 2048) == 773);
  CHECK(hash_opposite(s, 0x08080808, 256) == 5);
  const RhfgConfig c{14, 5, 6, 0x5eed};
  const uint32_t want[5] = {8155, 7898, 16351, 5467, 12273};
  for (uint32_t i = 0; i < 5; ++i) CHECK(rhfg(s, i, 0xC0A80101, c) == want[i]);
}

TEST_CASE("hash_opposite determinism and eta=1") {
  HashSeeds a(42), b(42), c(43);
  CHECK(hash_opposite(a, 0xdeadbeef, 1) == 0);
  CHECK(hash_opposite(a, 12345, 2048) == hash_opposite(b, 12345, 2048));
  bool diff = false;
  for (uint32_t x = 0; x < 64; ++x) diff |= hash_opposite(a, x, 2048) != hash_opposite(c, x, 2048);
  CHECK(diff);
}

TEST_CASE("rhfg rows, recover_block, blocks_consistent") {
  HashSeeds s(kPaper.seed);
  const uint32_t c0 = rhfg(s, 0, 0, kPaper);
  for (uint32_t i = 1; i < kPaper.r; ++i) CHECK(rhfg(s, i, 0, kPaper) == c0);
  CHECK(rhfg(s, 1, 0xffffffff, kPaper) == ((0x3fffu ^ rhfg(s, 0, 0xffffffff, kPaper)) & 0x3fff));
  CHECK_THROWS_AS(rhfg(s, kPaper.r, 1, kPaper), std::out_of_range);
  std::mt19937_64 rng(5);
  for (const RhfgConfig& cfg : {kPaper, kDesk}) {
    HashSeeds hs(cfg.seed);
    for (int t = 0; t < 20000; ++t) {
      const uint32_t cip = static_cast<uint32_t>(rng());
      const uint32_t col0 = rhfg(hs, 0, cip, cfg);
      for (uint32_t i = 1; i < cfg.r; ++i) REQUIRE(recover_block(col0, rhfg(hs, i, cip, cfg)) == slice(cip, i, cfg));
    }
  }
  CHECK(blocks_consistent(0, 0, kPaper));
  CHECK_FALSE(blocks_consistent(0x3f00, 0x0001, kPaper));
}

TEST_CASE("assemble_ip round trips and rejections") {
  std::vector<uint32_t> zeros(kPaper.r - 1, 0);
  CHECK(assemble_ip(zeros, kPaper) == 0u);
  std::mt19937_64 rng(7);
  for (const RhfgConfig& cfg : {kPaper, kDesk}) {
    HashSeeds hs(cfg.seed);
    for (int t = 0; t < 20000; ++t) {
      const uint32_t cip = static_cast<uint32_t>(rng());
      std::vector<uint32_t> b;
      const uint32_t col0 = rhfg(hs, 0, cip, cfg);
      for (uint32_t i = 1; i < cfg.r; ++i) b.push_back(recover_block(col0, rhfg(hs, i, cip, cfg)));
      REQUIRE(assemble_ip(b, cfg) == cip);
    }
  }
  std::vector<uint32_t> blocks(kDesk.r - 1, 0);
  blocks.back() = 1u << (kDesk.q - 1);
  CHECK_FALSE(assemble_ip(blocks, kDesk).has_value());
  CHECK_THROWS_AS(assemble_ip(std::vector<uint32_t>(2, 0), kDesk), std::invalid_argument);
}

TEST_CASE("validate_config diagnostics") {
  CHECK(validate_config(RhfgConfig{14, 5, 6, 0}, 2048, 300, 1024).empty());
  auto p = validate_config(RhfgConfig{8, 5, 6, 0}, 2048, 300, 1024);
  REQUIRE(!p.empty());
  CHECK(p.front().find("coverage") != std::string::npos);
  CHECK(validate_config(RhfgConfig{17, 5, 6, 0}, 2048, 300, 1024).front() == "q must be in [1, 16], got 17");
  CHECK(validate_config(RhfgConfig{14, 5, 6, 0}, 1, 300, 1024).front() == "eta must be >= 2, got 1");
  CHECK(validate_config(RhfgConfig{14, 5, 6, 0}, 2048, 0, 1024).front() == "k must be in [1, 65534], got 0");
}

TEST_CASE("estimator helpers") {
  SlidingEstimator se(8);
  for (Recorder v : se.recorders()) CHECK(v == kNeverSeen);
  se.touch(3);
  CHECK(se.recorders()[3] == 0);
  se.advance();
  CHECK(se.recorders()[3] == 1);
  CHECK(se.active_count(1) == 0);
  CHECK(se.active_count(2) == 1);
  CHECK_THROWS_AS(se.active_count(0), std::out_of_range);
  CHECK_THROWS_AS(se.touch(8), std::out_of_range);
  CHECK_THROWS_AS(SlidingEstimator(1), std::invalid_argument);
  SlidingEstimator sat(2);
  sat.touch(0);
  for (int i = 0; i < 65534; ++i) sat.advance();
  CHECK(sat.recorders()[0] == 65534);
  sat.advance();
  CHECK(sat.recorders()[0] == 65535);
  CHECK(hot_cutoff(2048, 1024) == 806);
  CHECK(hot_cutoff(256, 128) == 101);
  CHECK(std::fabs(estimate_cardinality(2048, 806) - 1024.0) < 1.0);
  CHECK(estimate_cardinality(2048, 2048) == 2048.0 * std::log(2048.0));
  SlidingEstimator a(4), b(4);
  a.touch(0);
  b.touch(1);
  b.touch(0);
  b.advance();
  CHECK(merge_min({a, b}).recorders()[0] == 0);
  CHECK(intersect_max({a, b}).recorders()[0] == 1);
  CHECK(intersect_max({a, b}).recorders()[1] == kNeverSeen);
  CHECK_THROWS_AS(merge_min({}), std::invalid_argument);
  CHECK_THROWS_AS(merge_min({SlidingEstimator(4), SlidingEstimator(5)}), std::invalid_argument);
}

TEST_CASE("worker_ranges U/V/W split") {
  const auto r = worker_ranges(10, 4);
  REQUIRE(r.size() == 4);
  CHECK((r[0] == std::pair<std::size_t, std::size_t>{0, 3}));
  CHECK((r[1] == std::pair<std::size_t, std::size_t>{3, 6}));
  CHECK((r[2] == std::pair<std::size_t, std::size_t>{6, 8}));
  CHECK((r[3] == std::pair<std::size_t, std::size_t>{8, 10}));
  CHECK(worker_ranges(5, 0).empty());
  std::mt19937_64 rng(110);
  for (int t = 0; t < 50; ++t) {
    const std::size_t q = rng() % 100000;
    const unsigned v = 1 + rng() % 64;
    const auto rr = worker_ranges(q, v);
    std::size_t lo = 0;
    for (unsigned i = 0; i < v; ++i) {
      CHECK(rr[i].first == lo);
      CHECK(rr[i].second - rr[i].first == q / v + (i < q % v ? 1 : 0));
      lo = rr[i].second;
    }
    CHECK(lo == q);
  }
}

TEST_CASE("ipv4 parsing and formatting") {
  CHECK(parse_ipv4("192.168.1.1") == 0xC0A80101u);
  CHECK(parse_ipv4("3232235777") == 0xC0A80101u);
  CHECK(format_ipv4(0xC0A80101u) == "192.168.1.1");
  CHECK_THROWS_AS(parse_ipv4("1.2.3"), std::invalid_argument);
  CHECK_THROWS_AS(parse_ipv4("1.2.3.256"), std::invalid_argument);
  CHECK_THROWS_AS(parse_ipv4("4294967296"), std::invalid_argument);
}

TEST_CASE("trace I/O round trips and errors") {
  std::vector<TraceRecord> recs{{0, 1, 2}, {0, 0xC0A80101u, 0x08080808u}, {5, 7, 9}};
  for (TraceFormat f : {TraceFormat::kBinary, TraceFormat::kText}) {
    std::stringstream ss;
    write_trace(recs, ss, f);
    CHECK(read_trace(ss, f) == recs);
  }
  std::stringstream empty;
  CHECK(read_trace(empty, TraceFormat::kBinary).empty());
  std::stringstream bad("XXXX\x01\0\0\0", std::ios::in | std::ios::binary);
  CHECK_THROWS_WITH_SUBSTR(read_trace(bad, TraceFormat::kBinary), "bad magic");
  std::stringstream regress("5,1.2.3.4,5.6.7.8\n4,1.2.3.4,5.6.7.8\n");
  CHECK_THROWS_WITH_SUBSTR(read_trace(regress, TraceFormat::kText), "timestamp regression at record 1");
  std::stringstream malformed("1,2\n");
  CHECK_THROWS_WITH_SUBSTR(read_trace(malformed, TraceFormat::kText), "malformed line 1");
  std::stringstream trunc;
  write_trace(recs, trunc, TraceFormat::kBinary);
  std::string t = trunc.str();
  t.pop_back();
  std::stringstream tr(t);
  CHECK_THROWS_WITH_SUBSTR(read_trace(tr, TraceFormat::kBinary), "truncated record at position 2");

  // parse_ipv4's forms, as trace.py mirrors them (tests/test_trace_io.py)
  std::stringstream forms("# c\n\n7, 16909060,+1.2.3.4.\n8,1.2.3.4,8.8.8.8\r\n");
  const std::vector<TraceRecord> want_forms{{7, 16909060u, 16909060u}, {8, 16909060u, 0x08080808u}};
  CHECK(read_trace(forms, TraceFormat::kText) == want_forms);
  for (const char* bad : {"1,1.2.3,4\n", "1,1.2.3.256,4\n", "1,1..2.3,4\n", "1,4294967296,4\n", "x,1,2\n",
                          "7,1.2.3.4.\r,1\n"}) {
    std::stringstream b(bad);
    CHECK_THROWS_WITH_SUBSTR(read_trace(b, TraceFormat::kText), "malformed line 1");
  }

  // traces longer than the reader's 65536-record blocks: exact round trip,
  // and error positions past a block boundary
  std::vector<TraceRecord> big(200003);
  for (std::size_t i = 0; i < big.size(); ++i)
    big[i] = {static_cast<uint32_t>(i / 7), static_cast<uint32_t>(i * 2654435761u), static_cast<uint32_t>(~i)};
  std::stringstream bs;
  write_trace(big, bs, TraceFormat::kBinary);
  CHECK(bs.str().size() == 8 + 12 * big.size());
  const std::string bytes = bs.str();
  std::stringstream bin(bytes);
  CHECK(read_trace(bin, TraceFormat::kBinary) == big);
  std::stringstream cut(bytes.substr(0, 8 + 12 * 65536 + 5));
  CHECK_THROWS_WITH_SUBSTR(read_trace(cut, TraceFormat::kBinary), "truncated record at position 65536");
  std::vector<TraceRecord> back(big);
  back[131073].ts = 0;
  std::stringstream rs;
  write_trace(back, rs, TraceFormat::kBinary);
  CHECK_THROWS_WITH_SUBSTR(read_trace(rs, TraceFormat::kBinary), "timestamp regression at record 131073");
}

TEST_CASE("orientation by core-network prefixes") {
  CnetSpec cnet({"10.0.0.0/8", "192.168.0.0/16"});
  CHECK(cnet.contains(0x0A010203));
  CHECK_FALSE(cnet.contains(0x0B000000));
  auto o = orient_pair(0x08080808, 0x0A000001, cnet);
  REQUIRE(o.has_value());
  CHECK(o->first == 0x0A000001u);
  CHECK_FALSE(orient_pair(0x0A000001, 0x0A000002, cnet).has_value());
  CHECK_THROWS_AS(CnetSpec({}), std::invalid_argument);
  CHECK_THROWS_AS(CnetSpec({"10.0.0.0"}), std::invalid_argument);
}

TEST_CASE("exact counts and synthetic truth") {
  WindowConfig win;
  win.k = 3;
  SynthSpec spec;
  spec.slots = 6;
  spec.planted.push_back({0x0A000001, 50, 1, 3});
  spec.background_hosts = 100;
  spec.pairs_per_slot = 300;
  spec.max_distinct_per_host = 8;
  const SynthResult res = synth_trace(spec, 9, win);
  const GroundTruth gt = exact_counts(res.trace, win);
  REQUIRE(gt.slots.size() == res.truth.slots.size());
  for (std::size_t s = 0; s < gt.slots.size(); ++s) CHECK(gt.slots[s] == res.truth.slots[s]);
  CHECK(gt.slots[1].at(0x0A000001) == 50);
  CHECK(gt.slots[5].at(0x0A000001) == 50);  // window 3..5 still holds slot 3
  SynthSpec none;
  none.slots = 0;
  CHECK_THROWS_AS(synth_trace(none, 1, win), std::invalid_argument);
  std::istringstream in("slots 4\nbackground hosts=10 pairs-per-slot=5\nsuper cip=10.0.0.1 count=7 from=1 to=2\n");
  const SynthSpec p = parse_synth_spec(in);
  CHECK(p.slots == 4);
  CHECK(p.background_hosts == 10);
  REQUIRE(p.planted.size() == 1);
  CHECK(p.planted[0].count == 7);
  std::istringstream bad("bogus\n");
  CHECK_THROWS_WITH_SUBSTR(parse_synth_spec(bad), "synth spec line 1: unknown stanza: bogus");
}

TEST_CASE("evaluate normalises by true super points") {
  std::unordered_map<uint32_t, uint32_t> truth{{1, 10}, {2, 3}, {3, 20}};
  auto r = evaluate({1, 2}, truth, 10);
  CHECK(r.fpr == 0.5);
  CHECK(r.fnr == 0.5);
  CHECK(r.tfr == 1.0);
  auto d = evaluate({5}, {{1, 1}}, 10);
  CHECK(d.degenerate);
  CHECK(d.fpr == 1.0);
}

#ifdef HAVE_REF
TEST_CASE("synth_trace equals the reference generator record for record") {
  for (uint64_t seed : {77ull, 104ull, 107ull}) {
    SynthSpec spec;
    spec.slots = 5;
    for (uint32_t i = 0; i < 3; ++i) spec.planted.push_back({0x0A000000 + i, 200, 0, 4});
    spec.background_hosts = 500;
    spec.pairs_per_slot = 700;
    spec.max_distinct_per_host = 8;
    WindowConfig win;
    win.k = 5;
    const auto ours = synth_trace(spec, seed, win).trace;
    std::vector<uint32_t> planted;
    for (const auto& p : spec.planted) planted.insert(planted.end(), {p.cip, p.count, p.slot_lo, p.slot_hi});
    const size_t n = ref_synth_trace(planted.data(), spec.planted.size(), 500, 1.1, 700, 8, 5, seed, 1.0, 5, 0,
                                     nullptr, 0);
    std::vector<uint32_t> recs(3 * n);
    ref_synth_trace(planted.data(), spec.planted.size(), 500, 1.1, 700, 8, 5, seed, 1.0, 5, 0, recs.data(), n);
    REQUIRE(ours.size() == n);
    for (size_t i = 0; i < n; ++i)
      REQUIRE((ours[i] == TraceRecord{recs[3 * i], recs[3 * i + 1], recs[3 * i + 2]}));
  }
}

// The text reader's canonical fast path (workload.cpp, parse_line_canonical)
// against the reference's reader: random lines, mostly well-formed, with
// signs, spaces, '\r', long numbers, extra fields and stray dots mixed in.
// Each trace must give the same records, or fail with the same message.
TEST_CASE("text read_trace equals the reference reader on random lines") {
  std::mt19937_64 rng(0x7e47);
  auto pick = [&rng](uint64_t n) { return rng() % n; };
  auto number = [&](bool octet) -> std::string {
    switch (pick(120)) {
      case 0: return std::to_string(rng());                       // long, may overflow
      case 1: return "+" + std::to_string(pick(300));
      case 2: return " " + std::to_string(pick(300));
      case 3: return "0" + std::to_string(pick(1000));
      case 4: return std::to_string(pick(300)) + "x";
      case 5: return "";
      default: return std::to_string(octet ? pick(256 + 4) : pick(uint64_t{1} << 33));
    }
  };
  auto ip = [&]() -> std::string {
    if (pick(4) == 0) return number(false);
    std::string s;
    const int n = pick(10) == 0 ? 3 + static_cast<int>(pick(3)) : 4;
    for (int i = 0; i < n; ++i) s += (i ? "." : "") + number(true);
    if (pick(20) == 0) s += ".";
    return s;
  };
  int parsed = 0;
  for (int trace = 0; trace < 3000; ++trace) {
    std::string text;
    uint32_t ts = 0;
    const int lines = 1 + static_cast<int>(pick(4));
    for (int l = 0; l < lines; ++l) {
      ts += static_cast<uint32_t>(pick(3));
      std::string line = pick(8) == 0 ? number(false) : std::to_string(ts);
      line += "," + ip() + "," + ip();
      if (pick(15) == 0) line += "," + ip();
      if (pick(15) == 0) line += "\r";
      if (pick(30) == 0) line = "# comment";
      if (pick(30) == 0) line.clear();
      text += line + "\n";
    }
    std::string ours_err, ref_err;
    std::vector<TraceRecord> ours;
    try {
      std::stringstream in(text);
      ours = read_trace(in, TraceFormat::kText);
    } catch (const std::exception& e) {
      ours_err = e.what();
    }
    std::vector<uint32_t> recs(3 * 16);
    size_t n = 0;
    if (ref_read_trace(text.data(), text.size(), 0, recs.data(), 16, &n) != 0) ref_err = ref_last_error();
    REQUIRE(ours_err == ref_err);
    if (!ref_err.empty()) continue;
    REQUIRE(ours.size() == n);
    for (size_t i = 0; i < n; ++i)
      REQUIRE((ours[i] == TraceRecord{recs[3 * i], recs[3 * i + 1], recs[3 * i + 2]}));
    ++parsed;
  }
  std::cerr << "  " << parsed << " of 3000 random traces parsed, the rest failed identically\n";
  CHECK(parsed > 300);
}

// validate_config's whole message list against the reference (hashing.cpp:63-87)
// over q 0..18, r 0..8, delta 0..q+1, four eta, k and theta values each:
// 120,384 cases, every one compared message for message.
TEST_CASE("validate_config equals the reference on the full grid") {
  const uint32_t etas[] = {0, 1, 2, 256};
  const uint32_t ks[] = {0, 1, 65534, 65535};
  const double thetas[] = {0, 0.5, 1, 1024};
  size_t cases = 0, flagged = 0;
  char buf[2048];
  for (uint32_t q = 0; q <= 18; ++q)
    for (uint32_t r = 0; r <= 8; ++r)
      for (uint32_t d = 0; d <= q + 1; ++d)
        for (uint32_t eta : etas)
          for (uint32_t k : ks)
            for (double th : thetas) {
              const auto ours = validate_config(RhfgConfig{q, r, d, 0}, eta, k, th);
              const size_t n = ref_validate_all(q, r, d, eta, k, th, buf, sizeof buf);
              std::string joined;
              for (size_t i = 0; i < ours.size(); ++i) joined += (i ? "\n" : "") + ours[i];
              if (ours.size() != n || joined != buf) {
                std::ostringstream os;
                os << "q=" << q << " r=" << r << " delta=" << d << " eta=" << eta << " k=" << k
                   << " theta=" << th << ": ours [" << joined << "] ref [" << buf << "]";
                FAIL(os.str());
              }
              ++cases;
              flagged += n != 0;
            }
  std::cerr << "  " << cases << " configurations, " << flagged << " with diagnostics, 0 differences\n";
  CHECK(cases == 120384);
  // the delta=0 case the CLI prints in full (tools/sspd.cpp:65-70)
  const auto d0 = validate_config(RhfgConfig{14, 5, 0, 0}, 2048, 5, 1024);
  REQUIRE(d0.size() == 2);
  CHECK(d0[1] == "address coverage (r-2)*delta+q = 14 < 32");
}

// assemble_ip / blocks_consistent (hashing.cpp:45-61, hashing.hpp:80-84) on
// random and adversarial blocks over every geometry validate_config accepts
// with r <= 12, against the reference.
TEST_CASE("assemble_ip and blocks_consistent equal the reference") {
  std::mt19937_64 rng(0xa55e);
  size_t geos = 0, accepted = 0, total = 0;
  for (uint32_t q = 1; q <= 16; ++q)
    for (uint32_t r = 3; r <= 12; ++r)
      for (uint32_t d = 1; d < q; ++d) {
        const RhfgConfig cfg{q, r, d, 0};
        if (!validate_config(cfg, 2, 1, 1).empty()) continue;
        ++geos;
        std::vector<uint32_t> b(r - 1);
        for (int t = 0; t < 400; ++t) {
          const uint32_t cip = static_cast<uint32_t>(rng());
          for (uint32_t i = 1; i < r; ++i) {
            b[i - 1] = ((cip >> (((i - 1) * d) & 31u)) & cfg.column_mask());
            if (t % 3 == 1) b[i - 1] ^= (rng() % 7 == 0) ? (1u << (rng() % q)) : 0;  // corrupt some
            if (t % 3 == 2) b[i - 1] = static_cast<uint32_t>(rng()) & cfg.column_mask();
          }
          uint32_t ip = 0;
          const int ref = ref_assemble_ip(q, r, d, b.data(), &ip);
          const auto ours = assemble_ip(b, cfg);
          REQUIRE(ours.has_value() == (ref != 0));
          if (ref) REQUIRE(*ours == ip);
          accepted += ref != 0;
          ++total;
          const uint32_t lo = static_cast<uint32_t>(rng()) & cfg.column_mask();
          const uint32_t hi = static_cast<uint32_t>(rng()) & cfg.column_mask();
          REQUIRE(blocks_consistent(lo, hi, cfg) == (ref_blocks_consistent(q, r, d, lo, hi) != 0));
          const uint32_t hi2 = (lo >> d) | (hi & ~((1u << (q - d)) - 1));
          REQUIRE(blocks_consistent(lo, hi2, cfg) == (ref_blocks_consistent(q, r, d, lo, hi2) != 0));
        }
      }
  std::cerr << "  " << geos << " geometries, " << total << " block lists (" << accepted << " assembled)\n";
  CHECK(geos > 300);
}

// hot_cutoff / estimate_cardinality (estimator.cpp:25-36): the same doubles
// and size_t bit for bit, over eta 1..4096 and random theta and R_k.
TEST_CASE("hot_cutoff and estimate_cardinality equal the reference") {
  std::mt19937_64 rng(0xc0f);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  size_t n = 0;
  for (size_t eta = 1; eta <= 4096; ++eta) {
    for (double th : {0.0, 1.0, 0.5 * eta, static_cast<double>(eta), 1024.0, 1e9, u(rng) * 4 * eta}) {
      REQUIRE(hot_cutoff(eta, th) == ref_hot_cutoff(eta, th));
      ++n;
    }
    for (size_t rk : {size_t{0}, size_t{1}, eta - 1, eta, static_cast<size_t>(rng() % eta)}) {
      const double a = estimate_cardinality(eta, rk), b = ref_estimate(eta, rk);
      REQUIRE(std::memcmp(&a, &b, sizeof a) == 0);
      ++n;
    }
  }
  for (size_t eta : {size_t{1} << 16, size_t{1} << 20, size_t{1} << 31})
    for (int t = 0; t < 2000; ++t) {
      const double th = u(rng) * 2.0 * static_cast<double>(eta);
      REQUIRE(hot_cutoff(eta, th) == ref_hot_cutoff(eta, th));
      const size_t rk = rng() % (eta + 1);
      const double a = estimate_cardinality(eta, rk), b = ref_estimate(eta, rk);
      REQUIRE(std::memcmp(&a, &b, sizeof a) == 0);
      n += 2;
    }
  std::cerr << "  " << n << " cutoffs and estimates, bit-identical\n";
}

// parse_ipv4 / format_ipv4 (workload.cpp:37-64): random strings give the
// same value, or the same exception type and message.
TEST_CASE("parse_ipv4 and format_ipv4 equal the reference") {
  std::mt19937_64 rng(0x1b4);
  auto pick = [&rng](uint64_t n) { return rng() % n; };
  const char* alphabet = "0123456789....  +-x\r\tabcdef";
  size_t ok = 0, n = 0;
  for (int t = 0; t < 200000; ++t) {
    std::string s;
    switch (pick(4)) {
      case 0:  // dotted quads, sometimes off by one field or octet
        for (int i = 0, m = 3 + static_cast<int>(pick(3)); i < m; ++i)
          s += (i ? "." : "") + std::to_string(pick(10) ? pick(256) : pick(100000));
        break;
      case 1:
        s = std::to_string(pick(4) ? pick(uint64_t{1} << 32) : rng());
        break;
      default:
        for (int i = 0, m = static_cast<int>(pick(12)); i < m; ++i) s += alphabet[pick(std::strlen(alphabet))];
    }
    int code = 0;
    uint32_t mine = 0;
    std::string err;
    try {
      mine = parse_ipv4(s);
    } catch (const std::invalid_argument& e) {
      code = 1, err = e.what();
    } catch (const std::out_of_range& e) {
      code = 2, err = e.what();
    } catch (const std::exception& e) {
      code = 3, err = e.what();
    }
    uint32_t theirs = 0;
    const int rc = ref_parse_ipv4(s.c_str(), &theirs);
    if (rc != code || (rc && err != ref_last_error()) || (!rc && mine != theirs))
      FAIL("parse_ipv4(\"" + s + "\"): ours " + std::to_string(code) + " " + err + " ref " +
                             std::to_string(rc) + " " + (rc ? ref_last_error() : ""));
    ok += rc == 0;
    ++n;
  }
  char buf[32];
  for (int t = 0; t < 100000; ++t) {
    const uint32_t ip = t < 16 ? (t & 1 ? ~0u << t : 1u << t) : static_cast<uint32_t>(rng());
    ref_format_ipv4(ip, buf, sizeof buf);
    REQUIRE(format_ipv4(ip) == buf);
  }
  std::cerr << "  " << n << " strings (" << ok << " parsed), 100000 formatted\n";
  CHECK(ok > 1000);
}

// parse_synth_spec (workload.cpp:302-358): random specs give the same spec,
// or the same message.
TEST_CASE("parse_synth_spec equals the reference") {
  std::mt19937_64 rng(0x5bec);
  auto pick = [&rng](uint64_t n) { return rng() % n; };
  auto num = [&]() -> std::string {
    switch (pick(16)) {
      case 0: return "x";
      case 1: return "";
      case 2: return std::to_string(rng());
      case 3: return "-" + std::to_string(pick(5));
      case 4: return "1e3";
      default: return std::to_string(pick(5000));
    }
  };
  size_t ok = 0;
  for (int t = 0; t < 20000; ++t) {
    std::string text;
    for (int l = 0, m = static_cast<int>(pick(6)); l < m; ++l) {
      switch (pick(8)) {
        case 0: text += "slots " + num(); break;
        case 1: text += "background hosts=" + num() + " zipf=" + (pick(2) ? "1.25" : num()) +
                        " pairs-per-slot=" + num() + " max-distinct=" + num(); break;
        case 2: text += "background " + std::string(pick(2) ? "hosts" : "zipf=0.9"); break;
        case 3: text += "super cip=" + std::string(pick(3) ? "10.0.0." + std::to_string(pick(300)) : num()) +
                        " count=" + num() + (pick(2) ? " from=" + num() : "") + (pick(2) ? " to=" + num() : ""); break;
        case 4: text += "super count=" + num(); break;
        case 5: text += pick(2) ? "# comment" : ""; break;
        case 6: text += "bogus a=b"; break;
        default: text += "super cip=1.2.3.4 count=" + num() + " extra"; break;
      }
      text += pick(10) ? "\n" : "\r\n";
    }
    std::string mine, err;
    int code = 0;
    try {
      std::istringstream in(text);
      const SynthSpec s = parse_synth_spec(in);
      char line[160];
      std::snprintf(line, sizeof line, "%u %u %a %u %u\n", s.slots, s.background_hosts, s.zipf_exponent,
                    s.pairs_per_slot, s.max_distinct_per_host);
      mine = line;
      for (const auto& p : s.planted) {
        std::snprintf(line, sizeof line, "%u %u %u %u\n", p.cip, p.count, p.slot_lo, p.slot_hi);
        mine += line;
      }
    } catch (const std::invalid_argument& e) {
      code = 1, err = e.what();
    } catch (const std::exception& e) {
      code = 3, err = e.what();
    }
    std::vector<char> out(1 << 16);
    const int rc = ref_parse_synth_spec(text.data(), text.size(), out.data(), out.size());
    if (rc != code || (rc ? err != ref_last_error() : mine != out.data()))
      FAIL("spec [" + text + "]: ours " + std::to_string(code) + " " + (code ? err : mine) +
                             " ref " + std::to_string(rc) + " " + (rc ? ref_last_error() : out.data()));
    ok += rc == 0;
  }
  std::cerr << "  20000 random specs (" << ok << " parsed)\n";
  CHECK(ok > 1000);
}
#endif

CHECK_MAIN
