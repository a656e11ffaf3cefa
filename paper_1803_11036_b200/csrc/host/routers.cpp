// Union-min run_detection over several GPUs in one process (routers.hpp).
#include "routers.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

#include "sspd/estimator.hpp"
#include "sspd_cuda.h"

namespace sspd::detail {
namespace {

void check(sspd_status st) {
  if (st == SSPD_OK) return;
  const std::string msg = sspd_last_error();
  if (st == SSPD_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == SSPD_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

}  // namespace

Routers::Routers(const RhfgConfig& cfg, uint32_t eta, uint32_t k_max, std::size_t candidate_cap,
                 const std::vector<int>& devices, uint64_t region_cap)
    : eta_(eta), cap_(candidate_cap), region_cap_(region_cap), dev_(devices) {
  const std::size_t n = devices.size();
  std::vector<int> distinct(devices);
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  if (distinct.size() > 1) check(sspd_enable_peer_access(static_cast<int>(distinct.size()), distinct.data()));
  grids_.assign(n, nullptr);
  in_a_.assign(n, nullptr);
  in_b_.assign(n, nullptr);
  table_a_.assign(n, nullptr);
  table_b_.assign(n, nullptr);
  try {
    const uint64_t inbox_bytes = n * region_cap * 8;
    for (std::size_t i = 0; i < n; ++i) {
      // a partial grid: only router i's cells (n == 1: all of them)
      check(sspd_grid_create_sharded(devices[i], cfg.q, cfg.r, cfg.delta, cfg.seed, eta, k_max,
                                     static_cast<uint32_t>(n), static_cast<uint32_t>(i), &grids_[i]));
      check(sspd_device_alloc(devices[i], inbox_bytes, &in_a_[i]));
      check(sspd_device_alloc(devices[i], inbox_bytes, &in_b_[i]));
      check(sspd_device_alloc(devices[i], n * sizeof(void*), &table_a_[i]));
      check(sspd_device_alloc(devices[i], n * sizeof(void*), &table_b_[i]));
    }
    for (std::size_t i = 0; i < n; ++i) {
      check(sspd_grid_copy(grids_[i], table_a_[i], in_a_.data(), n * sizeof(void*), 1));
      check(sspd_grid_copy(grids_[i], table_b_[i], in_b_.data(), n * sizeof(void*), 1));
      check(sspd_set_shard_relay(grids_[i], table_a_[i], table_b_[i], static_cast<uint32_t>(n),
                                 static_cast<uint32_t>(i), region_cap));
    }
  } catch (...) {
    release();
    throw;
  }
}

Routers::~Routers() { release(); }

uint32_t* Routers::scratch(uint64_t words) {
  if (words > scratch_words_) {
    if (scratch_) check(sspd_device_free(dev_[0], scratch_));
    scratch_ = nullptr;
    scratch_words_ = 0;
    check(sspd_device_alloc(dev_[0], words * 4, &scratch_));
    scratch_words_ = words;
  }
  return static_cast<uint32_t*>(scratch_);
}

void Routers::release() {
  if (scratch_) sspd_device_free(dev_[0], scratch_);
  scratch_ = nullptr;
  scratch_words_ = 0;
  for (std::size_t i = 0; i < grids_.size(); ++i) {
    if (grids_[i]) sspd_grid_destroy(grids_[i]);
    for (void* p : {in_a_[i], in_b_[i], table_a_[i], table_b_[i]})
      if (p) sspd_device_free(dev_[i], p);
    grids_[i] = nullptr;
    in_a_[i] = in_b_[i] = table_a_[i] = table_b_[i] = nullptr;
  }
}

void Routers::scan(std::size_t router, std::span<const IpPair> pairs) {
  if (pairs.empty()) return;
  check(sspd_scan(grids_[router], reinterpret_cast<const uint32_t*>(pairs.data()), pairs.size(), 0));
}

void Routers::scan_records(std::size_t router, std::span<const TraceRecord> records) {
  if (records.empty()) return;
  check(sspd_scan_records(grids_[router], reinterpret_cast<const uint32_t*>(records.data()), records.size(), 0));
}

std::vector<uint64_t> Routers::sent(std::size_t router) {
  uint64_t* dev = nullptr;
  check(sspd_shard_sent(grids_[router], &dev));
  std::vector<uint64_t> host(64);
  check(sspd_grid_copy(grids_[router], host.data(), dev, 64 * 8, 0));  // also waits for the router's work
  return host;
}

void Routers::merge() {
  const std::size_t n = grids_.size();
  // hop 1 done on every router (the copies synchronise each stream)
  std::vector<std::vector<uint64_t>> s(n);
  for (std::size_t i = 0; i < n; ++i) s[i] = sent(i);
  for (std::size_t po = 0; po < n; ++po) {
    std::vector<uint64_t> counts(n);
    for (std::size_t src = 0; src < n; ++src) {
      counts[src] = s[src][po];
      if (counts[src] > region_cap_) throw std::runtime_error("run_detection: router exchange region overflow");
    }
    check(sspd_shard_relay_regions(grids_[po], static_cast<const uint32_t*>(in_a_[po]), region_cap_, counts.data(),
                                   static_cast<uint32_t>(n)));
  }
  for (std::size_t i = 0; i < n; ++i) s[i] = sent(i);  // hop 2 counts, after every relay finished
  for (std::size_t dst = 0; dst < n; ++dst)
    for (std::size_t src = 0; src < n; ++src) {
      const uint64_t c = s[src][32 + dst];
      if (src == dst || c == 0) continue;
      if (c > region_cap_) throw std::runtime_error("run_detection: router exchange region overflow");
      const auto* base = static_cast<const uint32_t*>(in_b_[dst]) + 2 * src * region_cap_;
      check(sspd_shard_receive(grids_[dst], base, c));
    }
  for (sspd_grid* g : grids_) check(sspd_grid_synchronize(g));
}

DetectionReport Routers::reconstruct(uint32_t k, double theta) {
  const std::size_t n = grids_.size();
  const uint64_t cutoff = hot_cutoff(eta_, theta);
  // hot bits: OR over the routers, one kernel on router 0's device reading
  // every router's bits over NVLink, then each router takes the merged copy
  // (sspd_shard_hot returns with each router's bits complete)
  std::vector<uint32_t*> hot(n);
  uint64_t words = 0;
  for (std::size_t i = 0; i < n; ++i) check(sspd_shard_hot(grids_[i], k, cutoff, &hot[i], &words));
  std::vector<void*> stream(n);
  for (std::size_t i = 0; i < n; ++i) check(sspd_grid_stream(grids_[i], &stream[i]));
  uint32_t* merged = scratch(words);
  std::vector<const uint32_t*> srcs(hot.begin(), hot.end());
  check(sspd_reduce_words(dev_[0], srcs.data(), static_cast<uint32_t>(n), words, 0, merged, stream[0]));
  check(sspd_grid_synchronize(grids_[0]));  // every router's bits read before any is overwritten
  const uint32_t* one[1] = {merged};
  for (std::size_t i = 0; i < n; ++i)  // queued before shard_select on the router's own stream
    check(sspd_reduce_words(dev_[i], one, 1, words, 0, hot[i], stream[i]));
  // the same joins everywhere; survivor masks: AND over the routers
  uint64_t n_surv = 0, mwords = 0, ovf_count = 0;
  uint32_t ovf_level = 0;
  std::vector<uint32_t*> masks(n);
  for (std::size_t i = 0; i < n; ++i) {
    const sspd_status st =
        sspd_shard_select(grids_[i], k, cutoff, cap_, &n_surv, &masks[i], &mwords, &ovf_level, &ovf_count);
    if (st == SSPD_CANDIDATE_OVERFLOW) throw CandidateOverflow(ovf_level, ovf_count, cap_);
    check(st);
  }
  if (n_surv) {  // AND over the routers into router 0's masks (it reports)
    uint32_t* anded = scratch(mwords);
    std::vector<const uint32_t*> msrcs(masks.begin(), masks.end());
    check(sspd_reduce_words(dev_[0], msrcs.data(), static_cast<uint32_t>(n), mwords, 1, anded, stream[0]));
    const uint32_t* one[1] = {anded};
    check(sspd_reduce_words(dev_[0], one, 1, mwords, 1, masks[0], stream[0]));  // then shard_finish, same stream
  }
  // router 0 holds the merged masks: it reports
  std::vector<sspd_detection> buf(1024);
  DetectionReport rep;
  for (;;) {
    uint64_t got = 0;
    check(sspd_shard_finish(grids_[0], cutoff, buf.data(), buf.size(), &got));
    if (got > buf.size()) {
      buf.resize(got);
      continue;
    }
    for (uint64_t i = 0; i < got; ++i) rep.hosts.push_back({buf[i].cip, estimate_cardinality(eta_, buf[i].r_k)});
    break;
  }
  return rep;
}

void Routers::advance() {
  for (sspd_grid* g : grids_) check(sspd_advance(g, 1));
}

}  // namespace sspd::detail
