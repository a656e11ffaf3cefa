// sspd/rsea.hpp -- the reversible sliding estimator array (RSEA), resident
// on a B200.  Same public surface as the reference class
// (proj/include/sspd/rsea.hpp:14-114): callers written against the reference
// compile unchanged.  Storage lives in device memory behind the C ABI
// (include/sspd_cuda.h); cells() / estimator() hand out spans of a host
// mirror that is materialised on demand (u32 stamps -> u16 distances) and
// written back before the next device operation if it was handed out
// mutably.  update() calls are buffered on the host and scanned as one batch
// before anything observes the grid (scan is order- and batch-invariant, so
// this is exact).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <vector>

#include "sspd/estimator.hpp"
#include "sspd/hashing.hpp"
#include "sspd/workload.hpp"

struct sspd_grid;

namespace sspd {

struct IpPair {
  uint32_t cip;
  uint32_t oip;
};

struct HotSet {
  uint32_t row;
  std::vector<uint32_t> cols;
};

struct Detection {
  uint32_t cip;
  double estimate;
};

struct DetectionReport {
  uint64_t slot = 0;
  std::vector<Detection> hosts;
};

class CandidateOverflow : public std::runtime_error {
 public:
  CandidateOverflow(uint32_t level, std::size_t count, std::size_t cap);
  uint32_t level;
  std::size_t count;
};

// B200 extension: bits per recorder stamp.  32 keeps the full distances;
// 8 and 16 keep in-window counts exact for k <= window only (and hence hot
// sets, finalize and reconstruction), at 1/4 and 1/2 of the memory.  Narrow
// grids throw std::invalid_argument from cells()/estimator(), copies,
// merge_rseas and operator== (include/sspd_cuda.h sspd_grid_create_narrow).
struct StampWidth {
  uint32_t bits = 32;
  uint32_t window = 0;  // k_max; required for bits < 32
};

class Rsea {
 public:
  Rsea(const RhfgConfig& cfg, uint32_t eta);
  Rsea(const RhfgConfig& cfg, uint32_t eta, StampWidth width);  // B200 extension
  Rsea(const Rsea& other);
  Rsea(Rsea&& other) noexcept;
  Rsea& operator=(const Rsea& other);
  Rsea& operator=(Rsea&& other) noexcept;
  ~Rsea();

  const RhfgConfig& cfg() const { return cfg_; }
  uint32_t eta() const { return eta_; }
  const HashSeeds& seeds() const { return seeds_; }
  std::size_t recorder_count() const { return n_; }

  std::span<Recorder> estimator(uint32_t row, uint32_t col);
  std::span<const Recorder> estimator(uint32_t row, uint32_t col) const;
  std::span<const Recorder> cells() const;
  std::span<Recorder> cells();

  void update(uint32_t cip, uint32_t oip);
  void scan_batch(std::span<const IpPair> pairs, unsigned workers);
  void advance_slot(unsigned workers);
  std::vector<HotSet> hot_sets(uint32_t k, double theta) const;
  std::optional<Detection> finalize_candidate(std::span<const uint32_t> cols, uint32_t k,
                                              double theta) const;
  DetectionReport reconstruct_recursive(uint32_t k, double theta) const;
  DetectionReport reconstruct_leveled(uint32_t k, double theta, unsigned workers) const;

  void set_candidate_cap(std::size_t cap) { candidate_cap_ = cap; }
  std::size_t candidate_cap() const { return candidate_cap_; }

  bool operator==(const Rsea& other) const;

  // ---- B200 extensions (not in the reference) ----
  int device() const;
  // Scan pairs already resident on this grid's device (no host copy).
  void scan_device(const IpPair* device_pairs, std::size_t n);
  // Scan (ts, cip, oip) trace records as they are (ts ignored): no host-side
  // conversion to pairs (sspd_scan_records).
  void scan_records(std::span<const TraceRecord> records);
  // Keep per-cell in-window counts for windows up to k incrementally.
  void track_window(uint32_t k);
  // The underlying C-ABI handle (include/sspd_cuda.h).
  sspd_grid* handle() const;
  StampWidth stamp_width() const;
  // Queue reconstruct_leveled on the device and return at once; the next
  // collect_reconstruction() returns its report (sspd_reconstruct_async).
  // Scans and advances may be issued in between.
  void reconstruct_leveled_async(uint32_t k, double theta) const;
  DetectionReport collect_reconstruction() const;

 private:
  struct Uninitialised {};
  Rsea(Uninitialised, const RhfgConfig& cfg, uint32_t eta);
  void sync() const;          // flush mirror writes and buffered updates
  void load_mirror() const;   // device -> host distances
  DetectionReport reconstruct(uint32_t k, double theta, uint64_t cap) const;

  RhfgConfig cfg_;
  uint32_t eta_;
  HashSeeds seeds_;
  std::size_t n_ = 0;
  sspd_grid* h_ = nullptr;
  std::size_t candidate_cap_ = std::size_t{1} << 24;
  mutable std::vector<Recorder> mirror_;
  mutable bool mirror_valid_ = false;
  mutable bool mirror_dirty_ = false;
  mutable std::vector<IpPair> pending_;
  mutable std::unique_ptr<std::mutex> mu_;
  mutable std::size_t pending_cap_ = 0;  // candidate cap of the queued reconstruction
};

}  // namespace sspd
