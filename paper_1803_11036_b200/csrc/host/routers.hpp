// routers.hpp -- union-min run_detection over several GPUs in one process
// (internal to csrc/host; the multi-process equivalent is
// paper_1803_11036_b200/dist.py ShardExchange).
//
// Router i (one per GPU) owns a 1/N slice of the cells and keeps exact stamps
// only there.  Per slot: every router scans its shards' pairs and sends each
// new pair to its pair owner; pair owners dedup the routers' union for their
// share, stamp their own cells and relay each pair once to the other cell
// owners; cell owners stamp what arrives.  Reconstruction ORs the routers'
// hot bits and ANDs the survivors' bucket masks (include/sspd_cuda.h,
// "sharded routers") with one device kernel over the routers' buffers, read
// over NVLink (sspd_reduce_words).  Each router's grid is partial: it
// allocates only its own cells (sspd_grid_create_sharded), so N GPUs hold an
// N-times larger table.  The reports equal the union-min merged grid's.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "sspd/rsea.hpp"

namespace sspd::detail {

class Routers {
 public:
  // devices[i] hosts router i (repeats allowed: several routers on one GPU);
  // region_cap bounds the pairs any router sends to one other per hop.
  Routers(const RhfgConfig& cfg, uint32_t eta, uint32_t k_max, std::size_t candidate_cap,
          const std::vector<int>& devices, uint64_t region_cap);
  ~Routers();
  Routers(const Routers&) = delete;
  Routers& operator=(const Routers&) = delete;

  std::size_t size() const { return grids_.size(); }
  void scan(std::size_t router, std::span<const IpPair> pairs);
  void scan_records(std::size_t router, std::span<const TraceRecord> records);
  void merge();  // the two hops
  DetectionReport reconstruct(uint32_t k, double theta);
  void advance();

 private:
  std::vector<uint64_t> sent(std::size_t router);  // 64 counters: hop 1, then hop 2
  void release();

  uint32_t eta_;
  std::size_t cap_;  // candidate cap
  uint64_t region_cap_;
  std::vector<int> dev_;
  std::vector<sspd_grid*> grids_;
  std::vector<void*> in_a_, in_b_;        // router i's inboxes (N regions of region_cap pairs)
  std::vector<void*> table_a_, table_b_;  // per router: device arrays of every router's inbox
  void* scratch_ = nullptr;               // on router 0's device: merged hot bits / masks
  uint64_t scratch_words_ = 0;
  uint32_t* scratch(uint64_t words);
};

}  // namespace sspd::detail
