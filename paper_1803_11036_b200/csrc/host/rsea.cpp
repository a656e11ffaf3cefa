// sspd::Rsea over the C ABI (include/sspd_cuda.h).  The grid lives on a
// B200; this file only keeps the reference's C++ surface and semantics
// (proj/src/rsea.cpp): argument checks and exception types/messages, the
// host mirror behind cells()/estimator(), and buffering of single updates.
#include "sspd/rsea.hpp"

#include <cstdlib>
#include <limits>
#include <string>

#include "sspd/device.hpp"
#include "sspd_cuda.h"

namespace sspd {
namespace {

thread_local int t_device = -1;

int env_device() {
  const char* e = std::getenv("SSPD_DEVICE");
  return e ? std::atoi(e) : 0;
}

[[noreturn]] void raise(sspd_status st) {
  const std::string msg = sspd_last_error();
  switch (st) {
    case SSPD_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case SSPD_OUT_OF_RANGE:
      throw std::out_of_range(msg);
    default:
      throw std::runtime_error(msg);
  }
}

void check(sspd_status st) {
  if (st != SSPD_OK) raise(st);
}

}  // namespace

void set_device(int device) { t_device = device; }
int current_device() { return t_device >= 0 ? t_device : env_device(); }
int device_count() {
  int n = 0;
  return sspd_device_count(&n) == SSPD_OK ? n : 0;
}
std::vector<int> device_ordinals() {
  std::vector<int> out(64);
  int n = 0;
  if (sspd_device_ordinals(out.data(), static_cast<int>(out.size()), &n) != SSPD_OK) return {};
  out.resize(static_cast<std::size_t>(std::min<int>(n, 64)));
  return out;
}

CandidateOverflow::CandidateOverflow(uint32_t level_, std::size_t count_, std::size_t cap)
    : std::runtime_error("candidate buffer cap exceeded at level " + std::to_string(level_) + ": " +
                         std::to_string(count_) + " tuples, cap " + std::to_string(cap)),
      level(level_),
      count(count_) {}

Rsea::Rsea(Uninitialised, const RhfgConfig& cfg, uint32_t eta)
    : cfg_(cfg), eta_(eta), seeds_(cfg.seed), mu_(std::make_unique<std::mutex>()) {}

Rsea::Rsea(const RhfgConfig& cfg, uint32_t eta) : Rsea(Uninitialised{}, cfg, eta) {
  const auto problems = validate_config(cfg, eta, 1, 1.0);
  if (!problems.empty()) throw std::invalid_argument("Rsea: " + problems.front());
  n_ = std::size_t{cfg.r} * cfg.columns() * eta;
  check(sspd_grid_create(current_device(), cfg.q, cfg.r, cfg.delta, cfg.seed, eta, &h_));
}

Rsea::Rsea(const RhfgConfig& cfg, uint32_t eta, StampWidth width) : Rsea(Uninitialised{}, cfg, eta) {
  const auto problems = validate_config(cfg, eta, 1, 1.0);
  if (!problems.empty()) throw std::invalid_argument("Rsea: " + problems.front());
  n_ = std::size_t{cfg.r} * cfg.columns() * eta;
  if (width.bits == 32 && width.window == 0)
    check(sspd_grid_create(current_device(), cfg.q, cfg.r, cfg.delta, cfg.seed, eta, &h_));
  else
    check(sspd_grid_create_narrow(current_device(), cfg.q, cfg.r, cfg.delta, cfg.seed, eta, width.bits,
                                  width.window, &h_));
}

StampWidth Rsea::stamp_width() const {
  StampWidth w;
  check(sspd_grid_stamp_width(h_, &w.bits, &w.window));
  return w;
}

Rsea::Rsea(const Rsea& other) : Rsea(Uninitialised{}, other.cfg_, other.eta_) {
  other.sync();
  n_ = other.n_;
  candidate_cap_ = other.candidate_cap_;
  check(sspd_grid_clone(other.h_, -1, &h_));
}

Rsea::Rsea(Rsea&& other) noexcept
    : cfg_(other.cfg_),
      eta_(other.eta_),
      seeds_(other.seeds_),
      n_(other.n_),
      h_(other.h_),
      candidate_cap_(other.candidate_cap_),
      mirror_(std::move(other.mirror_)),
      mirror_valid_(other.mirror_valid_),
      mirror_dirty_(other.mirror_dirty_),
      pending_(std::move(other.pending_)),
      mu_(std::move(other.mu_)) {
  other.h_ = nullptr;
}

Rsea& Rsea::operator=(const Rsea& other) {
  if (this != &other) {
    Rsea tmp(other);
    *this = std::move(tmp);
  }
  return *this;
}

Rsea& Rsea::operator=(Rsea&& other) noexcept {
  if (this != &other) {
    if (h_) sspd_grid_destroy(h_);
    cfg_ = other.cfg_;
    eta_ = other.eta_;
    seeds_ = other.seeds_;
    n_ = other.n_;
    h_ = other.h_;
    candidate_cap_ = other.candidate_cap_;
    mirror_ = std::move(other.mirror_);
    mirror_valid_ = other.mirror_valid_;
    mirror_dirty_ = other.mirror_dirty_;
    pending_ = std::move(other.pending_);
    mu_ = std::move(other.mu_);
    other.h_ = nullptr;
  }
  return *this;
}

Rsea::~Rsea() {
  if (h_) sspd_grid_destroy(h_);
}

sspd_grid* Rsea::handle() const {
  sync();
  return h_;
}

int Rsea::device() const {
  int d = 0;
  check(sspd_grid_info(h_, nullptr, &d, nullptr));
  return d;
}

// Mirror writes go to the device first, then the updates buffered after
// them: the order the reference would have applied them in.
void Rsea::sync() const {
  std::lock_guard<std::mutex> lk(*mu_);
  if (mirror_dirty_) {
    check(sspd_put_distances(h_, mirror_.data(), 0, n_));
    mirror_dirty_ = false;
  }
  if (!pending_.empty()) {
    check(sspd_scan(h_, reinterpret_cast<const uint32_t*>(pending_.data()), pending_.size(), 0));
    pending_.clear();
  }
}

void Rsea::load_mirror() const {
  std::lock_guard<std::mutex> lk(*mu_);
  if (mirror_valid_) return;
  mirror_.resize(n_);
  check(sspd_get_distances(h_, mirror_.data(), 0, n_));
  mirror_valid_ = true;
}

std::span<const Recorder> Rsea::cells() const {
  sync();
  load_mirror();
  return {mirror_.data(), n_};
}

std::span<Recorder> Rsea::cells() {
  sync();
  load_mirror();
  mirror_dirty_ = true;  // the caller may write through the span
  return {mirror_.data(), n_};
}

std::span<Recorder> Rsea::estimator(uint32_t row, uint32_t col) {
  return cells().subspan((std::size_t{row} * cfg_.columns() + col) * eta_, eta_);
}

std::span<const Recorder> Rsea::estimator(uint32_t row, uint32_t col) const {
  return cells().subspan((std::size_t{row} * cfg_.columns() + col) * eta_, eta_);
}

// Rsea::update (rsea.cpp:29-38): buffered; also applied to a live mirror so
// spans handed out earlier see it, like the reference's in-place store.
void Rsea::update(uint32_t cip, uint32_t oip) {
  std::lock_guard<std::mutex> lk(*mu_);
  pending_.push_back({cip, oip});
  if (mirror_valid_) {
    const uint32_t bucket = hash_opposite(seeds_, oip, eta_);
    const uint32_t col0 = static_cast<uint32_t>(seeds_.row0_raw(cip)) & cfg_.column_mask();
    for (uint32_t row = 0; row < cfg_.r; ++row) {
      const uint32_t col = row == 0 ? col0 : rhfg_from_row0(row, cip, col0, cfg_);
      mirror_[(std::size_t{row} * cfg_.columns() + col) * eta_ + bucket] = 0;
    }
  }
  if (pending_.size() >= (std::size_t{1} << 20)) {
    // bound the buffer: hand a full batch to the device
    if (mirror_dirty_) {
      check(sspd_put_distances(h_, mirror_.data(), 0, n_));
      mirror_dirty_ = false;
    }
    check(sspd_scan(h_, reinterpret_cast<const uint32_t*>(pending_.data()), pending_.size(), 0));
    pending_.clear();
  }
}

void Rsea::scan_batch(std::span<const IpPair> pairs, unsigned workers) {
  if (workers == 0) throw std::invalid_argument("scan_batch: workers == 0");
  if (pairs.empty()) return;
  sync();
  static_assert(sizeof(IpPair) == 8, "IpPair must be two packed u32");
  check(sspd_scan(h_, reinterpret_cast<const uint32_t*>(pairs.data()), pairs.size(), 0));
  std::lock_guard<std::mutex> lk(*mu_);
  mirror_valid_ = false;
}

void Rsea::scan_records(std::span<const TraceRecord> records) {
  if (records.empty()) return;
  sync();
  check(sspd_scan_records(h_, reinterpret_cast<const uint32_t*>(records.data()), records.size(), 0));
  std::lock_guard<std::mutex> lk(*mu_);
  mirror_valid_ = false;
}

void Rsea::scan_device(const IpPair* device_pairs, std::size_t n) {
  sync();
  check(sspd_scan(h_, reinterpret_cast<const uint32_t*>(device_pairs), n, 1));
  std::lock_guard<std::mutex> lk(*mu_);
  mirror_valid_ = false;
}

void Rsea::advance_slot(unsigned workers) {
  if (workers == 0) throw std::invalid_argument("advance_slot: workers == 0");
  sync();
  check(sspd_advance(h_, 1));
  std::lock_guard<std::mutex> lk(*mu_);
  mirror_valid_ = false;
}

void Rsea::track_window(uint32_t k) {
  sync();
  check(sspd_track_window(h_, k));
}

std::vector<HotSet> Rsea::hot_sets(uint32_t k, double theta) const {
  sync();
  std::vector<uint32_t> cols(std::size_t{cfg_.r} * cfg_.columns());
  std::vector<uint32_t> counts(cfg_.r);
  check(sspd_hot_sets(h_, k, hot_cutoff(eta_, theta), cols.data(), counts.data()));
  std::vector<HotSet> out(cfg_.r);
  std::size_t pos = 0;
  for (uint32_t row = 0; row < cfg_.r; ++row) {
    out[row].row = row;
    out[row].cols.assign(cols.begin() + pos, cols.begin() + pos + counts[row]);
    pos += counts[row];
  }
  return out;
}

std::optional<Detection> Rsea::finalize_candidate(std::span<const uint32_t> cols, uint32_t k,
                                                  double theta) const {
  if (cols.size() < cfg_.r) throw std::invalid_argument("finalize_candidate: expected r columns");
  sync();
  uint8_t ok = 0;
  uint32_t cip = 0, rk = 0;
  check(sspd_finalize(h_, cols.data(), 1, k, hot_cutoff(eta_, theta), &ok, &cip, &rk));
  if (!ok) return std::nullopt;
  return Detection{cip, estimate_cardinality(eta_, rk)};
}

DetectionReport Rsea::reconstruct(uint32_t k, double theta, uint64_t cap) const {
  sync();
  std::vector<sspd_detection> buf(1024);
  for (;;) {
    uint64_t n = 0, ovf_count = 0;
    uint32_t ovf_level = 0;
    const sspd_status st = sspd_reconstruct(h_, k, hot_cutoff(eta_, theta), cap, buf.data(), buf.size(), &n,
                                            &ovf_level, &ovf_count);
    if (st == SSPD_CANDIDATE_OVERFLOW) throw CandidateOverflow(ovf_level, ovf_count, cap);
    check(st);
    if (n > buf.size()) {
      buf.resize(n);
      continue;
    }
    DetectionReport rep;
    rep.hosts.reserve(n);
    for (uint64_t i = 0; i < n; ++i) rep.hosts.push_back({buf[i].cip, estimate_cardinality(eta_, buf[i].r_k)});
    return rep;
  }
}

void Rsea::reconstruct_leveled_async(uint32_t k, double theta) const {
  sync();
  pending_cap_ = candidate_cap_;
  check(sspd_reconstruct_async(h_, k, hot_cutoff(eta_, theta), candidate_cap_));
}

DetectionReport Rsea::collect_reconstruction() const {
  std::vector<sspd_detection> buf(1024);
  for (;;) {
    uint64_t n = 0, ovf_count = 0;
    uint32_t ovf_level = 0;
    const sspd_status st = sspd_reconstruct_collect(h_, buf.data(), buf.size(), &n, &ovf_level, &ovf_count);
    if (st == SSPD_CANDIDATE_OVERFLOW) throw CandidateOverflow(ovf_level, ovf_count, pending_cap_);
    check(st);
    if (n > buf.size()) {  // the reports stay readable: read again
      buf.resize(n);
      continue;
    }
    DetectionReport rep;
    rep.hosts.reserve(n);
    for (uint64_t i = 0; i < n; ++i) rep.hosts.push_back({buf[i].cip, estimate_cardinality(eta_, buf[i].r_k)});
    return rep;
  }
}

DetectionReport Rsea::reconstruct_leveled(uint32_t k, double theta, unsigned workers) const {
  if (workers == 0) throw std::invalid_argument("reconstruct_leveled: workers == 0");
  return reconstruct(k, theta, candidate_cap_);
}

DetectionReport Rsea::reconstruct_recursive(uint32_t k, double theta) const {
  return reconstruct(k, theta, std::numeric_limits<uint64_t>::max());
}

bool Rsea::operator==(const Rsea& other) const {
  if (n_ != other.n_) return false;
  sync();
  other.sync();
  int eq = 0;
  check(sspd_equal(h_, other.h_, &eq));
  return eq != 0;
}

}  // namespace sspd
