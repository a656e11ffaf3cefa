// ref_shim.cpp -- C ABI over the COMPILED REFERENCE (namespace renamed to
// sspd_ref by -Dsspd=sspd_ref in oracle/Makefile).  TEST INFRASTRUCTURE
// ONLY: used by tests/golden/make_golden.py to pin the oracle, by the parity
// tests when oracle/_ref/ is present, and by bench.py's --impl reference /
// cpu_baseline legs.  Built into oracle/_ref/libsspd_ref.so; this file is
// ours, the reference sources are compiled where they lie.
#include <cstdint>
#include <algorithm>
#include <cstring>
#include <exception>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "sspd/hashing.hpp"
#include "sspd/estimator.hpp"
#include "sspd/pipeline.hpp"
#include "sspd/rsea.hpp"
#include "sspd/snapshot.hpp"
#include "sspd/workload.hpp"

using namespace sspd_ref;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_h1_raw(uint64_t seed, uint32_t key) { return HashSeeds(seed).h1_raw(key); }
uint64_t ref_row0_raw(uint64_t seed, uint32_t key) { return HashSeeds(seed).row0_raw(key); }
uint32_t ref_hash_opposite(uint64_t seed, uint32_t oip, uint32_t eta) {
  return hash_opposite(HashSeeds(seed), oip, eta);
}
// Batch variants (one HashSeeds for many keys).
void ref_hash_batch(uint64_t seed, const uint32_t* keys, size_t n, uint64_t* h1, uint64_t* row0) {
  HashSeeds s(seed);
  for (size_t i = 0; i < n; ++i) {
    h1[i] = s.h1_raw(keys[i]);
    row0[i] = s.row0_raw(keys[i]);
  }
}
int ref_rhfg_cols(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, const uint32_t* cips,
                  size_t n, uint32_t* cols /* n*r */) {
  try {
    RhfgConfig cfg{q, r, delta, seed};
    HashSeeds s(seed);
    for (size_t i = 0; i < n; ++i)
      for (uint32_t row = 0; row < r; ++row) cols[i * r + row] = rhfg(s, row, cips[i], cfg);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}
int ref_assemble_ip(uint32_t q, uint32_t r, uint32_t delta, const uint32_t* blocks, uint32_t* ip) {
  RhfgConfig cfg{q, r, delta, 0};
  auto v = assemble_ip(std::span<const uint32_t>(blocks, r - 1), cfg);
  if (!v) return 0;
  *ip = *v;
  return 1;
}
int ref_blocks_consistent(uint32_t q, uint32_t r, uint32_t delta, uint32_t lo, uint32_t hi) {
  return blocks_consistent(lo, hi, RhfgConfig{q, r, delta, 0});
}
size_t ref_hot_cutoff(size_t eta, double theta) { return hot_cutoff(eta, theta); }
double ref_estimate(size_t eta, size_t rk) { return estimate_cardinality(eta, rk); }
int ref_validate(uint32_t q, uint32_t r, uint32_t delta, uint32_t eta, uint32_t k, double theta,
                 char* msg, size_t len) {
  auto p = validate_config(RhfgConfig{q, r, delta, 0}, eta, k, theta);
  if (!p.empty() && msg && len) {
    std::strncpy(msg, p.front().c_str(), len - 1);
    msg[len - 1] = 0;
  }
  return static_cast<int>(p.size());
}

// Every diagnostic validate_config returns (hashing.cpp:63-87), joined by
// '\n' into msg; returns how many there are.
size_t ref_validate_all(uint32_t q, uint32_t r, uint32_t delta, uint32_t eta, uint32_t k, double theta,
                        char* msg, size_t len) {
  const auto p = validate_config(RhfgConfig{q, r, delta, 0}, eta, k, theta);
  std::string all;
  for (size_t i = 0; i < p.size(); ++i) all += (i ? "\n" : "") + p[i];
  if (msg && len) {
    std::strncpy(msg, all.c_str(), len - 1);
    msg[len - 1] = 0;
  }
  return p.size();
}

// export_snapshot (snapshot.cpp:36-68) of a reference grid: the whole
// stream's bytes into out (cap bytes); returns the size, or 0 on error.
size_t ref_export_snapshot(void* g, uint32_t k, uint32_t theta, uint64_t slot, uint32_t node_id, char* out,
                           size_t cap) {
  try {
    const auto* rs = static_cast<Rsea*>(g);
    SnapshotMeta m;
    m.seed = rs->cfg().seed;
    m.q = rs->cfg().q;
    m.r = rs->cfg().r;
    m.delta = rs->cfg().delta;
    m.eta = rs->eta();
    m.k = k;
    m.theta = theta;
    m.slot = slot;
    m.node_id = node_id;
    std::ostringstream os(std::ios::out | std::ios::binary);
    export_snapshot(*rs, m, os);
    const std::string b = os.str();
    if (b.size() <= cap) std::memcpy(out, b.data(), b.size());
    return b.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return 0;
  }
}

// parse_ipv4 (workload.cpp:37-58): 0 and *ip, or 1 (invalid_argument),
// 2 (out_of_range), 3 (other) with what() in ref_last_error().
int ref_parse_ipv4(const char* text, uint32_t* ip) {
  try {
    *ip = parse_ipv4(text);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::out_of_range& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}
void ref_format_ipv4(uint32_t ip, char* out, size_t len) {
  std::strncpy(out, format_ipv4(ip).c_str(), len - 1);
  out[len - 1] = 0;
}

// parse_synth_spec (workload.cpp:302-358) over an in-memory spec.  On success
// returns 0 and a canonical rendering of the spec in out ("slots bg zipf(%a)
// pps maxd" then "cip count lo hi" per planted host, one line each); on error
// 1 (invalid_argument) or 3 with what() in ref_last_error().
int ref_parse_synth_spec(const char* text, size_t len, char* out, size_t outlen) {
  try {
    std::istringstream in(std::string(text, len));
    const SynthSpec s = parse_synth_spec(in);
    char line[160];
    std::snprintf(line, sizeof line, "%u %u %a %u %u\n", s.slots, s.background_hosts, s.zipf_exponent,
                  s.pairs_per_slot, s.max_distinct_per_host);
    std::string all = line;
    for (const auto& p : s.planted) {
      std::snprintf(line, sizeof line, "%u %u %u %u\n", p.cip, p.count, p.slot_lo, p.slot_hi);
      all += line;
    }
    std::strncpy(out, all.c_str(), outlen - 1);
    out[outlen - 1] = 0;
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

void* ref_grid_create(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta) {
  try {
    return new Rsea(RhfgConfig{q, r, delta, seed}, eta);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void* ref_grid_clone(void* g) { return new Rsea(*static_cast<Rsea*>(g)); }
void ref_grid_destroy(void* g) { delete static_cast<Rsea*>(g); }
size_t ref_grid_size(void* g) { return static_cast<Rsea*>(g)->recorder_count(); }
void ref_update(void* g, uint32_t cip, uint32_t oip) { static_cast<Rsea*>(g)->update(cip, oip); }
void ref_scan(void* g, const uint32_t* pairs, size_t n, unsigned workers) {
  static_assert(sizeof(IpPair) == 8);
  static_cast<Rsea*>(g)->scan_batch(
      std::span<const IpPair>(reinterpret_cast<const IpPair*>(pairs), n), workers);
}
// The reference pipeline's alpha-sized scan_batch calls (pipeline.cpp:58-63).
void ref_scan_alpha(void* g, const uint32_t* pairs, size_t n, unsigned workers, size_t alpha) {
  auto* rs = static_cast<Rsea*>(g);
  const auto* p = reinterpret_cast<const IpPair*>(pairs);
  for (size_t i = 0; i < n; i += alpha)
    rs->scan_batch(std::span<const IpPair>(p + i, std::min(alpha, n - i)), workers);
}
void ref_advance(void* g, unsigned workers) { static_cast<Rsea*>(g)->advance_slot(workers); }
void ref_get_cells(void* g, uint16_t* out) {
  auto c = static_cast<Rsea*>(g)->cells();
  std::memcpy(out, c.data(), c.size() * 2);
}
void ref_get_cells_range(void* g, size_t offset, size_t count, uint16_t* out) {
  auto c = static_cast<Rsea*>(g)->cells();
  std::memcpy(out, c.data() + offset, count * 2);
}
void ref_set_cells(void* g, const uint16_t* in) {
  auto c = static_cast<Rsea*>(g)->cells();
  std::memcpy(c.data(), in, c.size() * 2);
}
size_t ref_hot_sets(void* g, uint32_t k, double theta, uint32_t* cols, uint32_t* counts) {
  auto hs = static_cast<Rsea*>(g)->hot_sets(k, theta);
  size_t t = 0;
  for (size_t i = 0; i < hs.size(); ++i) {
    counts[i] = static_cast<uint32_t>(hs[i].cols.size());
    for (uint32_t c : hs[i].cols) cols[t++] = c;
  }
  return t;
}
int ref_finalize(void* g, const uint32_t* cols, uint32_t k, double theta, uint32_t* cip,
                 double* est) {
  auto* rs = static_cast<Rsea*>(g);
  auto d = rs->finalize_candidate(std::span<const uint32_t>(cols, rs->cfg().r), k, theta);
  if (!d) return 0;
  *cip = d->cip;
  *est = d->estimate;
  return 1;
}
// Returns 0 ok (n_out written, up to cap_out rows), 3 overflow, 1 invalid.
int ref_reconstruct(void* g, int leveled, uint32_t k, double theta, unsigned workers, size_t cap,
                    uint32_t* cips, double* ests, size_t cap_out, size_t* n_out,
                    uint32_t* ovf_level, size_t* ovf_count) {
  auto* rs = static_cast<Rsea*>(g);
  try {
    rs->set_candidate_cap(cap);
    DetectionReport rep = leveled ? rs->reconstruct_leveled(k, theta, workers)
                                  : rs->reconstruct_recursive(k, theta);
    *n_out = rep.hosts.size();
    for (size_t i = 0; i < rep.hosts.size() && i < cap_out; ++i) {
      cips[i] = rep.hosts[i].cip;
      ests[i] = rep.hosts[i].estimate;
    }
    return 0;
  } catch (const CandidateOverflow& e) {
    *ovf_level = e.level;
    *ovf_count = e.count;
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}
void* ref_merge(void* const* grids, size_t n, int policy) {
  try {
    std::vector<const Rsea*> v;
    for (size_t i = 0; i < n; ++i) v.push_back(static_cast<const Rsea*>(grids[i]));
    return new Rsea(merge_rseas(v, policy == 0 ? MergePolicy::kUnionMin : MergePolicy::kPaperMax));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
int ref_grid_equal(void* a, void* b) { return *static_cast<Rsea*>(a) == *static_cast<Rsea*>(b); }

// run_detection over shards of (ts, cip, oip) records. Reports are written as
// parallel arrays (slot, cip, estimate); returns 0, 3 on overflow, 1 invalid.
int ref_run_detection(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta,
                      double mu, uint32_t k, uint32_t start, double theta, uint32_t alpha,
                      unsigned workers, int policy, int leveled, size_t cap,
                      const uint32_t* recs, const size_t* shard_off, size_t n_shards,
                      uint64_t* slots, uint32_t* cips, double* ests, size_t cap_out,
                      size_t* n_out, size_t* n_reports) {
  try {
    RunConfig rc;
    rc.cfg = RhfgConfig{q, r, delta, seed};
    rc.eta = eta;
    rc.window.mu = mu;
    rc.window.k = k;
    rc.window.start = start;
    rc.theta = theta;
    rc.alpha = alpha;
    rc.workers = workers;
    rc.policy = policy == 0 ? MergePolicy::kUnionMin : MergePolicy::kPaperMax;
    rc.strategy = leveled ? Strategy::kLeveled : Strategy::kRecursive;
    rc.candidate_cap = cap;
    std::vector<std::vector<TraceRecord>> shards(n_shards);
    for (size_t s = 0; s < n_shards; ++s)
      for (size_t i = shard_off[s]; i < shard_off[s + 1]; ++i)
        shards[s].push_back({recs[3 * i], recs[3 * i + 1], recs[3 * i + 2]});
    auto reps = run_detection(shards, rc);
    size_t t = 0;
    for (const auto& rep : reps)
      for (const auto& h : rep.hosts) {
        if (t < cap_out) {
          slots[t] = rep.slot;
          cips[t] = h.cip;
          ests[t] = h.estimate;
        }
        ++t;
      }
    *n_out = t;
    *n_reports = reps.size();
    return 0;
  } catch (const CandidateOverflow& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// synth_trace (workload.cpp:215-300) for fixtures: planted = (cip, count,
// lo, hi) quadruples. Returns the record count; fills recs (3 u32 each) up
// to cap_recs.
size_t ref_synth_trace(const uint32_t* planted, size_t n_planted, uint32_t bg_hosts, double zipf,
                       uint32_t pairs_per_slot, uint32_t max_distinct, uint32_t slots,
                       uint64_t seed, double mu, uint32_t k, uint32_t start, uint32_t* recs,
                       size_t cap_recs) {
  SynthSpec spec;
  for (size_t i = 0; i < n_planted; ++i)
    spec.planted.push_back({planted[4 * i], planted[4 * i + 1], planted[4 * i + 2],
                            planted[4 * i + 3]});
  spec.background_hosts = bg_hosts;
  spec.zipf_exponent = zipf;
  spec.pairs_per_slot = pairs_per_slot;
  spec.max_distinct_per_host = max_distinct;
  spec.slots = slots;
  WindowConfig win;
  win.mu = mu;
  win.k = k;
  win.start = start;
  auto res = synth_trace(spec, seed, win);
  for (size_t i = 0; i < res.trace.size() && i < cap_recs; ++i) {
    recs[3 * i] = res.trace[i].ts;
    recs[3 * i + 1] = res.trace[i].cip;
    recs[3 * i + 2] = res.trace[i].oip;
  }
  return res.trace.size();
}

// read_trace (workload.cpp:66-96) over an in-memory text or binary trace.
// Returns 0 and the record count in *n (records filled up to cap_recs), or 3
// with the reference's message in ref_last_error().
int ref_read_trace(const char* data, size_t len, int binary, uint32_t* recs, size_t cap_recs,
                   size_t* n) {
  try {
    std::istringstream in(std::string(data, len), std::ios::in | std::ios::binary);
    const auto t = read_trace(in, binary ? TraceFormat::kBinary : TraceFormat::kText);
    for (size_t i = 0; i < t.size() && i < cap_recs; ++i) {
      recs[3 * i] = t[i].ts;
      recs[3 * i + 1] = t[i].cip;
      recs[3 * i + 2] = t[i].oip;
    }
    *n = t.size();
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

}  // extern "C"
