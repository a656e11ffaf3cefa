// sspd_cuda.cu -- C ABI (include/sspd_cuda.h) over the sm_100a kernels in
// kernels.cuh.  Host orchestration only: argument checks with the
// reference's error texts, per-grid streams and scratch, chunked host->device
// copies, and the bits of reconstruction that are inherently host-side
// (dedup + sort of the reported hosts, estimate_cardinality in double).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sspd_cuda.h"
#include "kernels.cuh"
#include "synth.h"

#ifndef SSPD_SCAN_BLOCKS_PER_SM
#define SSPD_SCAN_BLOCKS_PER_SM 4  // one resident wave (profiles/r01_ab_scan_grid.md)
#endif

#include <omp.h>

using namespace sspd_dev;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

sspd_status fail(sspd_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CU(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(SSPD_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                       " at " #call);                                \
  } while (0)

// splitmix64 / TabulationHash / HashSeeds (hashing.cpp:8-34): the device
// tables must equal the reference's bit for bit.
uint64_t splitmix64(uint64_t& s) {
  s += 0x9e3779b97f4a7c15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void fill_tab(uint64_t t[4][256], uint64_t seed) {
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 256; ++j) t[i][j] = splitmix64(s);
}

HashTabs make_tabs(uint64_t seed) {
  HashTabs h;
  uint64_t s = seed;
  const uint64_t h1_seed = splitmix64(s);
  const uint64_t row0_seed = splitmix64(s);
  fill_tab(h.h1, h1_seed);
  fill_tab(h.row0, row0_seed);
  return h;
}

// validate_config (hashing.cpp:63-87), first diagnostic only.
std::string first_problem(uint32_t q, uint32_t r, uint32_t delta, uint32_t eta) {
  if (q < 1 || q > 16) return "q must be in [1, 16], got " + std::to_string(q);
  if (delta == 0 || delta >= q)
    return "delta must satisfy 0 < delta < q, got delta=" + std::to_string(delta) +
           " q=" + std::to_string(q);
  if (r < 3) return "r must be >= 3, got " + std::to_string(r);
  const uint32_t coverage = (r - 2) * delta + q;
  if (coverage < 32)
    return "address coverage (r-2)*delta+q = " + std::to_string(coverage) + " < 32";
  if (eta < 2) return "eta must be >= 2, got " + std::to_string(eta);
  return "";
}

struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
  uint64_t units;
};

// Device block cache.  A paper-geometry grid is ~1 GiB of stamps, pair set
// and staging, and cudaMalloc + cudaFree of that costs ~70 ms -- more than
// a whole run_detection of ten 1M-pair slots.  Blocks of >= 1 MiB go back to
// a per-device cache when freed (best fit within 25%, at most
// $SSPD_CACHE_BYTES per device, default 16 GiB; flushed when cudaMalloc runs
// out of memory, and by sspd_release_cached).  cudaFree synchronises the
// device; a cached free does the same unless the caller knows the block is
// idle, so a block never changes hands while a kernel still uses it.
class BlockCache {
 public:
  static BlockCache& get() {
    static BlockCache* c = new BlockCache();  // never destroyed: usable from atexit paths
    return *c;
  }
  cudaError_t alloc(void** p, size_t want) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t bytes = want < kMin ? want : (want + kMin - 1) / kMin * kMin;
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto& f = free_[dev];
      auto it = f.lower_bound(bytes);
      if (it != f.end() && it->first <= bytes + bytes / 4) {
        *p = it->second;
        cached_[dev] -= it->first;
        live_[*p] = {it->first, dev};
        f.erase(it);
        return cudaSuccess;
      }
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      release(dev);
      e = cudaMalloc(p, bytes);
    }
    if (e != cudaSuccess) {
      *p = nullptr;
      return e;
    }
    std::lock_guard<std::mutex> lk(mu_);
    live_[*p] = {bytes, dev};
    return cudaSuccess;
  }
  void free(void* p, bool idle) {
    if (!p) return;
    std::unique_lock<std::mutex> lk(mu_);
    auto it = live_.find(p);
    if (it == live_.end()) {
      lk.unlock();
      cudaFree(p);
      return;
    }
    const auto [bytes, dev] = it->second;
    live_.erase(it);
    if (bytes < kMin || cached_[dev] + bytes > cap_) {
      lk.unlock();
      cudaFree(p);
      return;
    }
    lk.unlock();
    if (!idle) {  // what cudaFree would have done: the block's device idles
      int cur = 0;
      cudaGetDevice(&cur);
      if (cur != dev) cudaSetDevice(dev);
      cudaDeviceSynchronize();
      if (cur != dev) cudaSetDevice(cur);
    }
    lk.lock();
    free_[dev].emplace(bytes, p);
    cached_[dev] += bytes;
  }
  // Free every cached block of `device` (-1: all devices).
  void release(int device) {
    std::vector<std::pair<int, void*>> out;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (auto& [dev, f] : free_) {
        if (device >= 0 && dev != device) continue;
        for (auto& [bytes, p] : f) out.emplace_back(dev, p);
        f.clear();
        cached_[dev] = 0;
      }
    }
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& [dev, p] : out) {
      cudaSetDevice(dev);
      cudaFree(p);
    }
    cudaSetDevice(cur);
  }
  uint64_t cached_bytes(int device) {
    std::lock_guard<std::mutex> lk(mu_);
    uint64_t t = 0;
    for (auto& [dev, b] : cached_)
      if (device < 0 || dev == device) t += b;
    return t;
  }

 private:
  BlockCache() {
    if (const char* e = std::getenv("SSPD_CACHE_BYTES")) cap_ = std::strtoull(e, nullptr, 10);
  }
  static constexpr size_t kMin = size_t{1} << 20;
  size_t cap_ = size_t{16} << 30;
  std::mutex mu_;
  std::map<int, std::multimap<size_t, void*>> free_;
  std::map<int, size_t> cached_;
  std::map<void*, std::pair<size_t, int>> live_;
};

// Pinned host buffers (scan staging of pageable input, small scratch):
// cudaMallocHost/cudaFreeHost cost milliseconds, so freed buffers are kept
// for reuse by exact size, up to 1 GiB in all.
class PinnedCache {
 public:
  static PinnedCache& get() {
    static PinnedCache* c = new PinnedCache();
    return *c;
  }
  cudaError_t alloc(void** p, size_t bytes) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto it = free_.find(bytes);
      if (it != free_.end()) {
        *p = it->second;
        cached_ -= bytes;
        free_.erase(it);
        live_[*p] = bytes;
        return cudaSuccess;
      }
    }
    cudaError_t e = cudaMallocHost(p, bytes);
    if (e != cudaSuccess) {
      *p = nullptr;
      return e;
    }
    std::lock_guard<std::mutex> lk(mu_);
    live_[*p] = bytes;
    return cudaSuccess;
  }
  // The caller guarantees no copy still reads or writes the buffer.
  void free(void* p) {
    if (!p) return;
    std::unique_lock<std::mutex> lk(mu_);
    auto it = live_.find(p);
    const size_t bytes = it == live_.end() ? 0 : it->second;
    if (it != live_.end()) live_.erase(it);
    if (bytes && cached_ + bytes <= (size_t{1} << 30)) {
      free_.emplace(bytes, p);
      cached_ += bytes;
      return;
    }
    lk.unlock();
    cudaFreeHost(p);
  }
  uint64_t release() {
    std::vector<void*> out;
    uint64_t n = 0;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (auto& [b, p] : free_) out.push_back(p);
      free_.clear();
      n = cached_;
      cached_ = 0;
    }
    for (void* p : out) cudaFreeHost(p);
    return n;
  }

 private:
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
  std::map<void*, size_t> live_;
  size_t cached_ = 0;
};

// Host worker threads for packing pageable input (scan_locked).  They sleep
// on a condition variable between regions: OpenMP's spinning workers stole
// the cores from the caller's own threads (profiles/r01_bench_api.md).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();
    return *p;
  }
  // fn(t, T) for t in [0, T) on T threads, the caller being thread 0.
  void run(unsigned T, const std::function<void(unsigned, unsigned)>& fn) {
    T = std::min<unsigned>(T, static_cast<unsigned>(n_workers_) + 1);
    if (T <= 1) {
      fn(0, 1);
      return;
    }
    std::lock_guard<std::mutex> one(call_mu_);  // one region at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      T_ = T;
      left_ = T - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0, T);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return left_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    n_workers_ = std::min(15u, hw - 1);
    for (unsigned i = 0; i < n_workers_; ++i) std::thread([this, i] { loop(i + 1); }).detach();
  }
  void loop(unsigned id) {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (id >= T_) continue;
      const auto* f = fn_;
      const unsigned T = T_;
      lk.unlock();
      (*f)(id, T);
      lk.lock();
      if (--left_ == 0) done_.notify_one();
    }
  }
  unsigned n_workers_ = 0;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  const std::function<void(unsigned, unsigned)>* fn_ = nullptr;
  unsigned T_ = 0, left_ = 0;
  uint64_t gen_ = 0;
};

cudaError_t cache_alloc(void** p, size_t bytes) { return BlockCache::get().alloc(p, bytes); }
void cache_free(void* p, bool idle = false) { BlockCache::get().free(p, idle); }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    cache_free(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cache_alloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release(bool idle = false) {
    cache_free(p, idle);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// DevBuf owned by one call: released on every exit path.
struct ScopedBuf : DevBuf {
  ScopedBuf() = default;
  ScopedBuf(const ScopedBuf&) = delete;
  ScopedBuf& operator=(const ScopedBuf&) = delete;
  ~ScopedBuf() { release(); }
};

}  // namespace

struct sspd_grid {
  int device = 0;
  uint32_t q = 0, r = 0, delta = 0, eta = 0;
  uint64_t seed = 0;
  Geo geo{};
  Div40 by_eta{};
  uint32_t now = kBaseNow;
  uint32_t* stamps = nullptr;
  uint32_t* touched = nullptr;
  uint64_t n_words = 0;  // bitmap words
  bool pending = false;  // touched has bits not folded into stamps
  uint32_t K = 0;        // tracked window (0 = off)
  uint32_t* hist = nullptr;
  bool hist_valid = false;
  bool pristine = true;  // every stamp still 0 (nothing scanned, imported or merged in)
  HashTabs* d_tabs = nullptr;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  DevBuf stage[2];       // host pair staging
  int stage_next = 0;    // the staging buffer the next host chunk goes to
  void* host_stage[2] = {nullptr, nullptr};  // pinned: pageable input packed here as pairs
  uint64_t host_stage_bytes = 0;
  cudaEvent_t ev_hcopy[2] = {nullptr, nullptr};  // the H2D out of host_stage[i] finished
  DevBuf stage_pairs[2]; // host trace records: their (cip, oip) pairs
  DevBuf rec_pairs;      // device trace records: their pairs
  DevBuf counts, hot_cols, hot_rowcnt, hotT, tupA, tupB, misc;
  DevBuf hot_words, hot_chunks;  // parallel hot compaction scratch
  DevBuf meta, surv;            // reconstruction bookkeeping, survivors
  ReconMeta* meta_host = nullptr;  // pinned mirror of meta
  uint64_t cap_alloc = 0;       // tuples per candidate buffer
  int scan_filter = 1;          // L1 duplicate filter in the scan (SSPD_SCAN_FILTER=0 disables)
  int scan_mode = -1;           // 0 bitmap, 1 direct, 2 dedup, 3 binned dedup, -1 auto
  DevBuf bin_counts, binned;    // binned dedup: per-(region, CTA) counts, partitioned pairs
  DevBuf pairset;               // dedup mode: per-slot set of seen (cip, oip) pairs
  bool shard = false;           // sharded routers (sspd_set_shard): own a 1/world slice of the cells
  ShardArgs shard_args{};       // one hop: to the cell owners; relayed: hop 1, to the pair owners
  bool relay = false;           // two hops (sspd_set_shard_relay)
  ShardArgs shard_b{};          // relayed: hop 2, pair owner -> cell owners
  DevBuf relayset;              // relayed: the pair owner's per-slot set of pairs it relayed
  bool relayset_dirty = false;
  DevBuf shard_sent;            // 2 x 32 u64: pairs pushed to each owner this slot (hop 1, hop 2)
  DevBuf shard_ovf;             // u32: a device-counted region ran past its stride
  DevBuf masks;                 // sharded reconstruction: per-survivor bucket masks
  DevBuf* last_tuples = nullptr;  // buffer holding the last reconstruction's r-tuples
  // sspd_reconstruct_async: one queued reconstruction awaiting collect
  bool recon_pending = false;
  cudaEvent_t ev_recon = nullptr;
  uint64_t pend_cutoff = 0, pend_cap = 0, pend_C = 0;
  std::vector<sspd_detection> collected;  // the last collect's reports (re-read with a larger buffer)
  bool collected_ready = false;
  uint64_t surv_cap = 0;          // tuple capacity the survivor arrays were laid out for
  uint64_t pairset_mask = 0;
  bool pairset_dirty = false;   // holds keys from the current slot
  bool record_touched = false;  // direct/dedup: also record the slot's bitmap (multi-router merge)
  bool export_pairs = false;    // dedup: also list the slot's distinct pairs (multi-router merge)
  DevBuf newpairs;              // this slot's distinct pairs (export_pairs)
  DevBuf newpairs_count;        // u64 on device
  uint64_t scanned_in_slot = 0; // pairs scanned since the last advance (list capacity bound)
  uint64_t list_pad_slots = 0;  // bound on the list blocks' padding since the last advance
  PushArgs push{};              // fused exchange: peer inboxes (export mode 3)
  // 8 KB of pinned memory.  The first 4 KB hold a queued reconstruction's
  // survivor prefix (2 x 512 u32) from recon_queue until it is collected; the
  // second 4 KB are scratch for synchronous counter/flag read-backs
  // (pinned_scratch), which may run while a reconstruction is pending.
  void* pinned_small = nullptr;
  // partial grid (sspd_grid_create_sharded): only cells [geo.own_lo,
  // geo.own_hi) are allocated, at stamps_alloc; `stamps` is based so that
  // recorder i of an owned cell is still stamps[i]
  bool partial = false;
  uint32_t part_world = 1, part_rank = 0;
  uint32_t* stamps_alloc = nullptr;
  bool profiling = false;
  int prof_suspend = 0;  // inside a PDL launch chain: one event pair around the chain only
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> event_pool;  // recycled profiling events (creation is the costly part)
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic, for e2e accounting
  // narrow stamps (width 8 or 16, kernels.cuh "NARROW STAMPS"): `codes`
  // replaces `stamps`, the window ring (K = k_max) is always on, and codes
  // are rebased before code(now) passes code_hi
  uint32_t width = 32;
  void* codes = nullptr;
  uint32_t code_lo = 0, code_hi = 0;
  uint32_t epoch0 = 0;  // code(now) = code_lo + (now - epoch0)
  // 16-bit scan: load the recorders before the atomics, so the atomics hit
  // L2 (C2 at 40 GiB: 4.19 vs 4.76 ms/slot, profiles/r01_ab_narrow_preload.md);
  // SSPD_NARROW_PRELOAD=0 turns it off
  bool narrow_preload = true;
  // Pipelined dedup scan (kernels.cuh scan_dedup_pipe_kernel) for the
  // window-ring path: -1 off (scan_dedup_kernel), 0 on, 1 on with L2
  // eviction priorities.  $SSPD_DEDUP_PIPE overrides (A/B runs).
  int dedup_pipe = 0;
  DevBuf fresh_count;  // u64: pairs new to their slot, summed over the pipelined scans
  // Compact key set (kernels.cuh scan_cset_kernel): 2^cset_lg u32 entries
  // keyed by (cip, bucket), the default for the pipelined path when
  // eta <= 2^16.  $SSPD_CSET=0 turns it off, $SSPD_CSET_LOG2 sizes it.
  int use_cset = 1;
  int cset_hint = 1;            // L2 priorities in the key-set scan ($SSPD_CSET_HINT=0: off)
  int cset8 = 1;                // 8-bit grids' dedup on the key-set scan too ($SSPD_CSET8=0: the narrow scan)
  uint32_t cset_pass_log2 = 0;  // 2^k passes per batch, each over 1/2^k of the set ($SSPD_CSET_PASSES)
  DevBuf cset;
  uint32_t cset_lg = 0;         // log2 entries of the (next) allocation
  bool cset_dirty = false;
  bool cset_fixed = false;      // $SSPD_CSET_LOG2 given: no growth
  // growth: the fresh-key counter is copied to pinned memory at each slot
  // end and read one advance later (no host wait), so the set is sized from
  // the keys a slot actually produced
  unsigned long long* cset_pin = nullptr;
  cudaEvent_t cset_ev = nullptr;
  bool cset_ev_pending = false;
  uint64_t cset_seen_total = 0;
  uint32_t cset_seen_now = 0, cset_pin_now = 0;
  uint32_t code_now() const { return code_lo + (now - epoch0); }
  std::mutex mu;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

int sm_count(int dev) {
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  n = n > 0 ? n : 148;
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

// Persistent-style grid size: a multiple of the SM count.
unsigned grid_blocks(const sspd_grid* g, uint64_t work_items, unsigned threads, unsigned per_sm) {
  const uint64_t need = (work_items + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sm_count(g->device) * per_sm;
  return (unsigned)std::max<uint64_t>(1, std::min(need, cap));
}

cudaEvent_t take_event(sspd_grid* g) {
  cudaEvent_t e = nullptr;
  if (!g->event_pool.empty()) {
    e = g->event_pool.back();
    g->event_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  return e;
}

struct Prof {
  sspd_grid* g;
  ProfRec rec{};
  bool on = false;
  // counts_launch: false for a span of several launches counted on their own
  Prof(sspd_grid* g_, const char* name, uint64_t units, bool counts_launch = true) : g(g_) {
    if (counts_launch) g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g->profiling || g->prof_suspend) return;
    on = true;
    rec.name = name;
    rec.units = units;
    rec.a = take_event(g);
    rec.b = take_event(g);
    cudaEventRecord(rec.a, g->stream);
  }
  ~Prof() {
    if (!on) return;
    cudaEventRecord(rec.b, g->stream);
    g->prof.push_back(rec);
  }
};

// Entry points that need the full 32-bit stamps (distances, merges,
// exchanges) refuse narrow grids instead of returning inexact data.
// Calls that need every cell's stamps on this grid.
sspd_status whole_only(const sspd_grid* g, const char* what) {
  if (!g->partial) return SSPD_OK;
  return fail(SSPD_INVALID_ARGUMENT, std::string(what) + ": a sharded router's partial grid holds only cells " +
                                         std::to_string(g->geo.own_lo) + ".." + std::to_string(g->geo.own_hi - 1) +
                                         " (use the shard calls)");
}

sspd_status wide_only(const sspd_grid* g, const char* what) {
  if (g->width == 32) return SSPD_OK;
  return fail(SSPD_INVALID_ARGUMENT, std::string(what) + ": not available on a grid with " +
                                         std::to_string(g->width) + "-bit stamps (exact for in-window counts "
                                         "with k <= " + std::to_string(g->K) + " only)");
}

// Counter/flag read-back scratch, disjoint from the survivor prefix.
void* pinned_scratch(const sspd_grid* g) { return static_cast<char*>(g->pinned_small) + 4096; }

sspd_status no_pending(const sspd_grid* g, const char* what) {
  if (!g->recon_pending) return SSPD_OK;
  return fail(SSPD_INVALID_ARGUMENT, std::string(what) + ": a queued reconstruction awaits sspd_reconstruct_collect");
}

sspd_status check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SSPD_CUDA_ERROR, std::string("CUDA launch: ") + cudaGetErrorString(e));
  return SSPD_OK;
}

// Launch with programmatic stream serialization: the kernel may begin while
// its predecessor in the stream finishes, and waits for the predecessor's
// results at its pdl_wait() (kernels.cuh).  Used along the reconstruction
// chain, whose kernels are each a few microseconds long.
template <class... KArgs, class... Args>
sspd_status launch_pdl(sspd_grid* g, void (*kernel)(KArgs...), unsigned grid, unsigned block, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = g->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return fail(SSPD_CUDA_ERROR, std::string("CUDA launch: ") + cudaGetErrorString(e));
  return SSPD_OK;
}

// The touched bitmap (1 bit per recorder: 2.7 GB at C2) exists only once a
// bitmap scan, a recorded exchange or sspd_grid_touched needs it; the dedup
// and direct scans never do.
sspd_status ensure_touched_locked(sspd_grid* g) {
  if (g->touched) return SSPD_OK;
  if (cache_alloc((void**)&g->touched, g->n_words * 4) != cudaSuccess) {
    cudaGetLastError();
    g->touched = nullptr;
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory allocating the touched bitmap");
  }
  CU(cudaMemsetAsync(g->touched, 0, g->n_words * 4, g->stream));
  return SSPD_OK;
}

sspd_status commit_locked(sspd_grid* g) {
  if (!g->pending) return SSPD_OK;
  const bool use_hist = g->K && g->hist_valid;
  const unsigned threads = 256;
  const unsigned blocks = grid_blocks(g, (g->n_words + 31) / 32 * 32, threads, 8);
  {
    Prof p(g, "commit", g->n_words);
    commit_kernel<<<blocks, threads, 0, g->stream>>>(g->touched, g->n_words, g->stamps, g->geo.n_rec,
                                                     g->now, use_hist ? g->hist : nullptr, g->K,
                                                     g->geo.ncells, g->by_eta);
  }
  g->pending = false;  // a stale window ring is rebuilt on demand
  return check_launch();
}

// The pair set may only skip a pair whose recorders still read `now`; any
// write to the stamps other than a scan invalidates it.
sspd_status pairset_reset_locked(sspd_grid* g) {
  if (!g->pairset_dirty && !g->cset_dirty) return SSPD_OK;
  if (g->pairset.p) CU(cudaMemsetAsync(g->pairset.p, 0xff, (g->pairset_mask + 1) * 8, g->stream));
  if (g->cset_dirty) CU(cudaMemsetAsync(g->cset.p, 0, (4ull << g->cset_lg), g->stream));
  g->pairset_dirty = g->cset_dirty = false;
  return SSPD_OK;
}

sspd_status hist_rebuild_locked(sspd_grid* g) {
  if (!g->K || g->hist_valid) return SSPD_OK;
  CU(cudaMemsetAsync(g->hist, 0, (size_t)g->K * g->geo.ncells * 4, g->stream));
  const unsigned blocks = grid_blocks(g, (uint64_t)g->geo.ncells * 32, 256, 8);
  {
    Prof p(g, "hist_rebuild", g->geo.ncells);
    hist_rebuild_kernel<<<blocks, 256, 0, g->stream>>>(g->stamps, g->geo, g->now, g->K, g->hist);
  }
  g->hist_valid = true;
  return check_launch();
}

// Per-cell R_k into g->counts (device).
sspd_status counts_locked(sspd_grid* g, uint32_t k) {
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (g->counts.ensure((size_t)g->geo.ncells * 4) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (counts)");
  if (k == 0 || k > 0xFFFFu) {
    // distance < 0 never holds; distance < k > 65535 always holds (estimator.hpp:26-31)
    const unsigned blocks = grid_blocks(g, g->geo.ncells, 256, 4);
    Prof p(g, "fill", g->geo.ncells);
    fill_u32_kernel<<<blocks, 256, 0, g->stream>>>(g->counts.as<uint32_t>(), g->geo.ncells,
                                                   k == 0 ? 0u : g->eta);
  } else if (g->width != 32 && k > g->K) {
    return fail(SSPD_INVALID_ARGUMENT, "active_count: k = " + std::to_string(k) + " exceeds the window K = " +
                                           std::to_string(g->K) + " of a " + std::to_string(g->width) +
                                           "-bit grid");
  } else if (g->K && k <= g->K) {
    s = hist_rebuild_locked(g);
    if (s) return s;
    const unsigned blocks = grid_blocks(g, g->geo.ncells, 256, 4);
    Prof p(g, "hist_counts", g->geo.ncells);
    hist_counts_kernel<<<blocks, 256, 0, g->stream>>>(g->hist, g->K, g->geo.ncells, g->now, k,
                                                      g->counts.as<uint32_t>());
  } else {
    const unsigned blocks = grid_blocks(g, (uint64_t)g->geo.ncells * 32, 256, 8);
    Prof p(g, "count", g->geo.ncells);
    count_kernel<<<blocks, 256, 0, g->stream>>>(g->stamps, g->geo, g->now - k,
                                                g->counts.as<uint32_t>());
  }
  return check_launch();
}

uint32_t words_per_key(const sspd_grid* g) {
  const uint32_t bits = 1u << g->delta;
  return bits <= 32 ? 1u : bits / 32u;
}

// Hot compaction into g->hot_cols / hot_rowcnt / hotT (device); row counts
// copied to host_rowcnt (synchronises).
// from_words: the hot bits are already in g->hot_words (OR-merged across
// sharded routers); only the transposed bits, chunk counts and compaction
// are rebuilt from them.
sspd_status hot_locked(sspd_grid* g, uint32_t k, uint64_t cutoff, std::vector<uint32_t>* host_rowcnt,
                       uint32_t* d_rowcnt, bool from_words = false, unsigned long long* zero = nullptr,
                       uint32_t zero_words = 0) {
  sspd_status s = SSPD_OK;
  // R_k straight from the window ring inside hot_mark when it covers k;
  // otherwise per-cell counts first (full pass over the stamps).
  const bool ring = !from_words && k >= 1 && k <= 0xFFFFu && g->K && k <= g->K;
  if (!from_words) {
    s = commit_locked(g);
    if (s) return s;
    s = ring ? hist_rebuild_locked(g) : counts_locked(g, k);
    if (s) return s;
  }
  const uint32_t ncol = 1u << g->q;
  const uint32_t chunks = (ncol + kHotChunk - 1) / kHotChunk;
  const uint32_t wpk = words_per_key(g);
  const size_t t_words = (size_t)g->r * ((size_t)wpk << (g->q - g->delta));
  if (g->hot_cols.ensure((size_t)g->r * ncol * 4) != cudaSuccess ||
      g->hot_rowcnt.ensure((size_t)g->r * 4) != cudaSuccess || g->hotT.ensure(t_words * 4) != cudaSuccess ||
      g->hot_words.ensure((size_t)g->r * ((ncol + 31) / 32) * 4) != cudaSuccess ||
      g->hot_chunks.ensure((size_t)g->r * chunks * 4) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (hot sets)");
  if (!d_rowcnt) d_rowcnt = g->hot_rowcnt.as<uint32_t>();
  {
    Prof p(g, "hot_compact", g->geo.ncells);
    hot_mark_kernel<<<g->r * chunks, kHotChunk, 0, g->stream>>>(
        g->counts.as<uint32_t>(), ring ? g->hist : nullptr, g->K, g->now, k, g->geo, cutoff,
        g->hot_words.as<uint32_t>(), g->hot_chunks.as<uint32_t>(), from_words ? 1 : 0, zero, zero_words);
    s = check_launch();
    if (s) return s;
    s = launch_pdl(g, hot_write_kernel, g->r * chunks, kHotChunk, g->hot_words.as<uint32_t>(), g->geo,
                   g->hot_chunks.as<uint32_t>(), g->hot_cols.as<uint32_t>(), d_rowcnt, g->hotT.as<uint32_t>(), wpk);
    if (s) return s;
  }
  if (host_rowcnt) {
    host_rowcnt->resize(g->r);
    CU(cudaMemcpyAsync(host_rowcnt->data(), d_rowcnt, g->r * 4, cudaMemcpyDeviceToHost, g->stream));
    g->d2h_bytes += g->r * 4;
    CU(cudaStreamSynchronize(g->stream));
  }
  return SSPD_OK;
}

// estimate_cardinality (estimator.cpp:25-30), host double arithmetic.
double estimate(uint64_t eta, uint64_t r_k) {
  const uint64_t z0 = eta - r_k;
  const double deta = static_cast<double>(eta);
  if (z0 == 0) return deta * std::log(deta);
  return -deta * std::log(static_cast<double>(z0) / deta);
}

int kmode_of(uint32_t k) { return k == 0 ? 1 : (k > 0xFFFFu ? 2 : 0); }

// Survivor buffers for up to n tuples.
sspd_status ensure_surv(sspd_grid* g, uint64_t n) {
  if (g->surv.ensure((size_t)std::max<uint64_t>(n, 1) * 12) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (finalize)");
  return SSPD_OK;
}

// Queue finalize_check + finalize_count over the r-tuples in `tuples`, their
// count taken from meta->level[r-1] (device).
sspd_status queue_finalize(sspd_grid* g, const uint32_t* tuples, uint64_t in_cap, uint32_t k) {
  uint32_t* s_idx = g->surv.as<uint32_t>();
  uint32_t* s_cip = s_idx + in_cap;
  uint32_t* s_rk = s_cip + in_cap;
  ReconMeta* meta = g->meta.as<ReconMeta>();
  sspd_status s;
  {
    Prof p(g, "finalize_check", in_cap, false);  // launch_pdl counts the launch
    s = launch_pdl(g, finalize_check_kernel, grid_blocks(g, in_cap, 256, 2), 256, tuples, in_cap,
                   (const HashTabs*)g->d_tabs, g->geo, meta, s_idx, s_cip, s_rk);
  }
  if (s) return s;
  {
    const uint32_t chunks = (g->eta + 1023) / 1024;
    const unsigned blocks = (unsigned)sm_count(g->device) * 8;
    Prof p(g, "finalize", in_cap * chunks, false);
    // live codes younger than k: code > code(now) - k, and never 0
    const uint32_t thr = (uint32_t)std::max<int64_t>((int64_t)g->code_now() - (k <= 0xFFFFu ? k : 0u),
                                                     (int64_t)g->code_lo - 1);
    const ReconMeta* cmeta = meta;
    const uint32_t* cidx = s_idx;
    if (g->width == 8)
      s = launch_pdl(g, finalize_count_narrow_kernel<uint8_t>, blocks, 256, tuples,
                     static_cast<const uint8_t*>(g->codes), g->geo, thr, kmode_of(k), cmeta, cidx, s_rk);
    else if (g->width == 16)
      s = launch_pdl(g, finalize_count_narrow_kernel<uint16_t>, blocks, 256, tuples,
                     static_cast<const uint16_t*>(g->codes), g->geo, thr, kmode_of(k), cmeta, cidx, s_rk);
    else
      s = launch_pdl(g, finalize_count_kernel, blocks, 256, tuples, (const uint32_t*)g->stamps, g->geo,
                     g->now - (k <= 0xFFFFu ? k : 0u), kmode_of(k), cmeta, cidx, s_rk);
  }
  return s;
}

// The per-slot pair set (dedup and shard scans), allocated on first use.
sspd_status ensure_pairset_locked(sspd_grid* g) {
  if (g->pairset.p) return SSPD_OK;
  // 8 B per exact key, a power of two of entries (SSPD_PAIRSET_LOG2,
  // default 2^25 = 256 MiB: ~10M distinct pairs per C2 slot at load 0.3;
  // measured 2^22..2^25 = 4.23..3.90 ms/slot, profiles/r01_ab_pairset.txt).
  // Pinning it in L2 with an access-policy window measured slower (same file).
  // sharded routers also keep what peers push to them (~2.4x their own new
  // pairs at N=8 on C2): twice the entries from 4 routers up
  uint32_t lg = g->shard && g->shard_args.world >= 4 ? 26 : 25;
  if (const char* e = std::getenv("SSPD_PAIRSET_LOG2")) lg = std::min(30, std::max(16, std::atoi(e)));
  const uint64_t entries = 1ull << lg;
  if (g->pairset.ensure(entries * 8) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (pair set)");
  g->pairset_mask = entries - 1;
  CU(cudaMemsetAsync(g->pairset.p, 0xff, entries * 8, g->stream));
  if (!g->fresh_count.p) {
    if (g->fresh_count.ensure(8) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
    CU(cudaMemsetAsync(g->fresh_count.p, 0, 8, g->stream));
  }
  return SSPD_OK;
}

// The compact key set, allocated on first use: 2^24 entries (64 MiB) keep
// a C2 slot's ~9.4M keys at load 0.56; $SSPD_CSET_LOG2 in [24, 30].
sspd_status ensure_cset_locked(sspd_grid* g) {
  if (!g->fresh_count.p) {
    if (g->fresh_count.ensure(8) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
    CU(cudaMemsetAsync(g->fresh_count.p, 0, 8, g->stream));
  }
  if (g->cset.p) return SSPD_OK;
  if (!g->cset_lg) {
    g->cset_lg = kCsetStartLog2;
    if (const char* e = std::getenv("SSPD_CSET_LOG2")) {
      g->cset_lg = std::min<uint32_t>(kCsetMaxLog2, std::max<uint32_t>(kCsetMinLog2, (uint32_t)std::atoi(e)));
      g->cset_fixed = true;
    }
  }
  if (g->cset.ensure(4ull << g->cset_lg) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (key set)");
  CU(cudaMemsetAsync(g->cset.p, 0, 4ull << g->cset_lg, g->stream));
  // $SSPD_L2_SETASIDE_MIB: the device's persisting-L2 set-aside, the
  // carve-out the set's evict_last probes may occupy (A/B knob; the driver
  // default is 0, capped at persistingL2CacheMaxSize)
  if (const char* e = std::getenv("SSPD_L2_SETASIDE_MIB")) {
    int maxb = 0;
    CU(cudaDeviceGetAttribute(&maxb, cudaDevAttrMaxPersistingL2CacheSize, g->device));
    const size_t want = std::min<size_t>((size_t)std::max(0, std::atoi(e)) << 20, (size_t)maxb);
    CU(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
    size_t got = 0;
    CU(cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize));
    std::fprintf(stderr, "[sspd] L2 set-aside %zu B (max %d B)\n", got, maxb);
  }
  return SSPD_OK;
}

// At a slot end (before the set is cleared): read the fresh-key count the
// previous slot end copied out, if that copy has landed, and grow the set for
// the coming slots when a slot's keys loaded it past kCsetMaxLoad; then copy
// this slot end's count.  Growth reallocates (the cleared set starts empty).
sspd_status cset_slot_end_locked(sspd_grid* g) {
  if (!g->cset.p || g->cset_fixed) return SSPD_OK;
  if (!g->cset_pin) {
    if (PinnedCache::get().alloc(reinterpret_cast<void**>(&g->cset_pin), 64) != cudaSuccess)
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of pinned memory");
    CU(cudaEventCreateWithFlags(&g->cset_ev, cudaEventDisableTiming));
  }
  if (g->cset_ev_pending) {
    if (cudaEventQuery(g->cset_ev) != cudaSuccess) return SSPD_OK;  // not landed yet: try at the next slot end
    g->cset_ev_pending = false;
    const uint64_t total = *g->cset_pin;
    if (g->cset_seen_now && g->cset_pin_now > g->cset_seen_now) {
      const uint64_t per_slot = (total - g->cset_seen_total) / (g->cset_pin_now - g->cset_seen_now);
      const uint64_t cap = 1ull << g->cset_lg;
      uint32_t lg = g->cset_lg;
      if ((double)per_slot > kCsetMaxLoad * (double)cap) {
        while (lg < kCsetMaxLog2 && (double)per_slot > kCsetMaxLoad * (double)(1ull << lg)) ++lg;
      } else {
        // shrink back (to at most 4x the load) once slots need far less: the
        // per-slot clear and the L2 footprint scale with the table
        while (lg > kCsetStartLog2 && (double)per_slot < kCsetMinLoad * (double)(1ull << lg)) --lg;
      }
      if (lg != g->cset_lg) {
        g->cset.release();
        g->cset_lg = lg;
        g->cset_dirty = false;
        // allocate (and clear) now, at the slot end, not inside the next scan
        if (sspd_status es = ensure_cset_locked(g)) return es;
      }
    }
    g->cset_seen_total = total;
    g->cset_seen_now = g->cset_pin_now;
  }
  CU(cudaMemcpyAsync(g->cset_pin, g->fresh_count.p, 8, cudaMemcpyDeviceToHost, g->stream));
  CU(cudaEventRecord(g->cset_ev, g->stream));
  g->cset_ev_pending = true;
  g->cset_pin_now = g->now + 1;  // the count covers every slot before now + 1
  return SSPD_OK;
}

bool compatible(const sspd_grid* a, const sspd_grid* b) {
  return a->seed == b->seed && a->q == b->q && a->r == b->r && a->delta == b->delta && a->eta == b->eta;
}

}  // namespace

extern "C" {

int sspd_abi_version(void) { return 1; }

const char* sspd_last_error(void) { return g_err.c_str(); }

uint64_t sspd_launch_count(void) { return g_launches.load(); }

sspd_status sspd_device_alloc(int device, uint64_t bytes, void** ptr) {
  *ptr = nullptr;
  DeviceGuard dg(device);
  if (cache_alloc(ptr, std::max<uint64_t>(bytes, 16)) != cudaSuccess) {
    cudaGetLastError();
    *ptr = nullptr;
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory allocating " + std::to_string(bytes) + " bytes");
  }
  return SSPD_OK;
}

sspd_status sspd_device_free(int device, void* ptr) {
  DeviceGuard dg(device);
  cache_free(ptr);
  return SSPD_OK;
}

sspd_status sspd_release_cached(int device, uint64_t* released) {
  BlockCache& c = BlockCache::get();
  if (released) *released = c.cached_bytes(device);
  c.release(device);
  const uint64_t pinned = PinnedCache::get().release();
  if (released) *released += pinned;
  return SSPD_OK;
}

sspd_status sspd_enable_peer_access(int n_devices, const int* devices) {
  for (int i = 0; i < n_devices; ++i)
    for (int j = 0; j < n_devices; ++j) {
      if (devices[i] == devices[j]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devices[i], devices[j]);
      if (!can) return fail(SSPD_CUDA_ERROR, "no peer access between devices " + std::to_string(devices[i]) +
                                                 " and " + std::to_string(devices[j]));
      DeviceGuard dg(devices[i]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(SSPD_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
  return SSPD_OK;
}

sspd_status sspd_grid_copy(sspd_grid* g, void* dst, const void* src, uint64_t bytes, int to_device) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (bytes == 0) return SSPD_OK;
  CU(cudaMemcpyAsync(dst, src, bytes, to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  if (to_device) g->h2d_bytes += bytes;
  else g->d2h_bytes += bytes;
  return SSPD_OK;
}

sspd_status sspd_device_ordinals(int* out, int cap, int* n) {
  int c = 0;
  *n = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return fail(SSPD_NO_DEVICE, "no CUDA device");
  }
  for (int d = 0; d < c; ++d) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    if (major != 10) continue;
    if (*n < cap && out) out[*n] = d;
    ++*n;
  }
  if (!*n) return fail(SSPD_NO_DEVICE, "no sm_100 device visible");
  return SSPD_OK;
}

sspd_status sspd_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess || c == 0) {
    cudaGetLastError();
    *n = 0;
    return fail(SSPD_NO_DEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  int ok = 0;
  for (int d = 0; d < c; ++d) {
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d);
    if (major == 10) ++ok;
  }
  *n = ok;
  if (!ok) return fail(SSPD_NO_DEVICE, "no sm_100 device visible");
  return SSPD_OK;
}

namespace {

sspd_status create_impl(int device, uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta,
                        uint32_t width, uint32_t k_max, sspd_grid** out, uint32_t part_world = 1,
                        uint32_t part_rank = 0) {
  *out = nullptr;
  const std::string prob = first_problem(q, r, delta, eta);
  if (!prob.empty()) return fail(SSPD_INVALID_ARGUMENT, "Rsea: " + prob);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(SSPD_NO_DEVICE, "sspd: no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= ndev) return fail(SSPD_INVALID_ARGUMENT, "sspd: bad device ordinal");
  DeviceGuard dg(device);
  auto* g = new sspd_grid();
  g->device = device;
  g->q = q;
  g->r = r;
  g->delta = delta;
  g->eta = eta;
  g->seed = seed;
  g->geo.q = q;
  g->geo.r = r;
  g->geo.delta = delta;
  g->geo.eta = eta;
  g->geo.col_mask = (1u << q) - 1u;
  g->geo.low_mask = (1u << (q - delta)) - 1u;
  g->geo.ncells = r << q;
  g->geo.n_rec = (uint64_t)g->geo.ncells * eta;
  // owned cells: those with shard_owner(c) == rank, i.e. c * world / ncells == rank
  g->geo.own_lo = (uint32_t)(((uint64_t)part_rank * g->geo.ncells + part_world - 1) / part_world);
  g->geo.own_hi = (uint32_t)(((uint64_t)(part_rank + 1) * g->geo.ncells + part_world - 1) / part_world);
  g->partial = part_world > 1;
  g->part_world = part_world;
  g->part_rank = part_rank;
  const uint64_t own_rec = (uint64_t)(g->geo.own_hi - g->geo.own_lo) * eta;
  g->by_eta = Div40::make(eta);
  g->width = width;
  if (const char* f = std::getenv("SSPD_SCAN_FILTER")) g->scan_filter = std::atoi(f) != 0;
  if (const char* f = std::getenv("SSPD_NARROW_PRELOAD")) g->narrow_preload = std::atoi(f) != 0;
  if (const char* f = std::getenv("SSPD_DEDUP_PIPE")) g->dedup_pipe = std::atoi(f);
  if (const char* f = std::getenv("SSPD_CSET")) g->use_cset = std::atoi(f);
  if (const char* f = std::getenv("SSPD_CSET_HINT")) g->cset_hint = std::atoi(f);
  if (const char* f = std::getenv("SSPD_CSET8")) g->cset8 = std::atoi(f);
  if (const char* f = std::getenv("SSPD_CSET_PASSES")) {
    const int v = std::atoi(f);
    g->cset_pass_log2 = v >= 4 ? 2 : v >= 2 ? 1 : 0;
  }
  // Device-resident pairs: deferred bitmap, measured faster than direct
  // stamping at both geometries (profiles/r01_ab_scan_modes.txt).
  if (const char* m = std::getenv("SSPD_SCAN_MODE")) {
    if (!std::strcmp(m, "bitmap")) g->scan_mode = 0;
    if (!std::strcmp(m, "direct")) g->scan_mode = 1;
    if (!std::strcmp(m, "dedup")) g->scan_mode = 2;
    if (!std::strcmp(m, "binned")) g->scan_mode = 3;
  }
  g->n_words = (g->geo.n_rec + 31) / 32;
  auto cleanup = [&](const std::string& why) {
    sspd_grid_destroy(g);
    return fail(SSPD_CUDA_ERROR, why);
  };
  if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup("CUDA error: stream creation failed");
  cudaEventCreateWithFlags(&g->ev_recon, cudaEventDisableTiming);
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&g->ev_copy[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_used[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_hcopy[i], cudaEventDisableTiming);
  }
  if (width != 32) {
    // narrow codes (all 0: nothing seen) and the always-on window ring
    const uint64_t bytes = g->geo.n_rec * (width / 8);
    if (cache_alloc((void**)&g->codes, bytes) != cudaSuccess) {
      cudaGetLastError();
      return cleanup("CUDA error: out of memory allocating " + std::to_string(bytes) + " bytes of stamps");
    }
    // u16 codes are positive normal bf16 bit patterns (the packed-bf16 max
    // atomic orders them like integers); u8 codes are plain bytes
    g->code_lo = width == 16 ? 0x0080u : 1u;
    g->code_hi = width == 16 ? 0x7F7Fu : 255u;
    g->epoch0 = g->now;
    g->K = k_max;
    if (cache_alloc((void**)&g->hist, (size_t)g->K * g->geo.ncells * 4) != cudaSuccess) {
      cudaGetLastError();
      return cleanup("CUDA error: out of memory (window ring)");
    }
    if (cudaMemsetAsync(g->codes, 0, bytes, g->stream) != cudaSuccess ||
        cudaMemsetAsync(g->hist, 0, (size_t)g->K * g->geo.ncells * 4, g->stream) != cudaSuccess)
      return cleanup("CUDA error: grid init");
    g->hist_valid = true;
  } else if (cache_alloc((void**)&g->stamps_alloc, own_rec * 4) != cudaSuccess) {
    cudaGetLastError();
    g->stamps_alloc = nullptr;
    return cleanup("CUDA error: out of memory allocating " + std::to_string(own_rec * 4) + " bytes of stamps");
  } else {
    g->stamps = g->stamps_alloc - (uint64_t)g->geo.own_lo * eta;
  }
  if (cache_alloc((void**)&g->d_tabs, sizeof(HashTabs)) != cudaSuccess) return cleanup("CUDA error: tables");
  if (PinnedCache::get().alloc(&g->pinned_small, 8192) != cudaSuccess ||
      PinnedCache::get().alloc(reinterpret_cast<void**>(&g->meta_host), sizeof(ReconMeta)) != cudaSuccess ||
      g->meta.ensure(sizeof(ReconMeta)) != cudaSuccess)
    return cleanup("CUDA error: pinned scratch");
  HashTabs h = make_tabs(seed);
  if (cudaMemcpyAsync(g->d_tabs, &h, sizeof h, cudaMemcpyHostToDevice, g->stream) != cudaSuccess)
    return cleanup("CUDA error: table upload");
  // All recorders never seen: stamp 0.
  if (width == 32 && cudaMemsetAsync(g->stamps_alloc, 0, own_rec * 4, g->stream) != cudaSuccess)
    return cleanup("CUDA error: grid init");
  if (cudaStreamSynchronize(g->stream) != cudaSuccess) return cleanup("CUDA error: grid init sync");
  *out = g;
  return SSPD_OK;
}

}  // namespace

sspd_status sspd_grid_create(int device, uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta,
                             sspd_grid** out) {
  return create_impl(device, q, r, delta, seed, eta, 32, 0, out);
}

sspd_status sspd_grid_create_sharded(int device, uint32_t q, uint32_t r, uint32_t delta, uint64_t seed,
                                     uint32_t eta, uint32_t k_max, uint32_t world, uint32_t rank, sspd_grid** out) {
  *out = nullptr;
  if (world < 1 || world > 32 || rank >= world)
    return fail(SSPD_INVALID_ARGUMENT, "create_sharded: need 1 <= world <= 32 and rank < world");
  if (k_max > 65534) return fail(SSPD_INVALID_ARGUMENT, "k must be in [1, 65534], got " + std::to_string(k_max));
  sspd_status s = create_impl(device, q, r, delta, seed, eta, 32, 0, out, world, rank);
  if (s || !k_max) return s;
  s = sspd_track_window(*out, k_max);
  if (s) {
    sspd_grid_destroy(*out);
    *out = nullptr;
  }
  return s;
}

sspd_status sspd_grid_owned(const sspd_grid* g, uint64_t* rec_lo, uint64_t* rec_hi) {
  *rec_lo = (uint64_t)g->geo.own_lo * g->eta;
  *rec_hi = (uint64_t)g->geo.own_hi * g->eta;
  return SSPD_OK;
}

sspd_status sspd_grid_create_narrow(int device, uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta,
                                    uint32_t width, uint32_t k_max, sspd_grid** out) {
  *out = nullptr;
  if (width != 8 && width != 16 && width != 32)
    return fail(SSPD_INVALID_ARGUMENT, "stamp width must be 8, 16 or 32, got " + std::to_string(width));
  if (k_max < 1 || k_max > 65534)
    return fail(SSPD_INVALID_ARGUMENT, "k must be in [1, 65534], got " + std::to_string(k_max));
  // an epoch of codes holds hi - lo - K + 2 slots; keep it >= 2
  if ((width == 8 && k_max > 254) || (width == 16 && k_max > 32511))
    return fail(SSPD_INVALID_ARGUMENT, "window k = " + std::to_string(k_max) + " needs more than " +
                                           std::to_string(width) + "-bit stamps");
  if (width == 32) {
    sspd_status s = create_impl(device, q, r, delta, seed, eta, 32, 0, out);
    if (s) return s;
    s = sspd_track_window(*out, k_max);
    if (s) {
      sspd_grid_destroy(*out);
      *out = nullptr;
    }
    return s;
  }
  return create_impl(device, q, r, delta, seed, eta, width, k_max, out);
}

sspd_status sspd_grid_stamp_width(const sspd_grid* g, uint32_t* width, uint32_t* k_max) {
  if (width) *width = g->width;
  if (k_max) *k_max = g->K;
  return SSPD_OK;
}

sspd_status sspd_grid_destroy(sspd_grid* g) {
  if (!g) return SSPD_OK;
  {
    DeviceGuard dg(g->device);
    // peers may still read this grid (merges, relays): the whole device
    // idles before its blocks go back to the cache
    cudaDeviceSynchronize();
    for (void* p : {(void*)g->stamps_alloc, (void*)g->codes, (void*)g->touched, (void*)g->hist, (void*)g->d_tabs})
      cache_free(p, true);
    PinnedCache::get().free(g->pinned_small);
    if (g->cset_pin) PinnedCache::get().free(g->cset_pin);
    if (g->cset_ev) cudaEventDestroy(g->cset_ev);
    PinnedCache::get().free(g->meta_host);
    for (int i = 0; i < 2; ++i) {
      PinnedCache::get().free(g->host_stage[i]);
      if (g->ev_hcopy[i]) cudaEventDestroy(g->ev_hcopy[i]);
    }
    for (DevBuf* b : {&g->stage[0], &g->stage[1], &g->stage_pairs[0], &g->stage_pairs[1], &g->rec_pairs, &g->counts, &g->hot_cols, &g->hot_rowcnt, &g->hotT,
                      &g->tupA, &g->tupB, &g->misc, &g->meta, &g->surv, &g->pairset, &g->newpairs,
                      &g->newpairs_count, &g->bin_counts, &g->binned, &g->hot_words, &g->hot_chunks, &g->relayset,
                      &g->shard_sent, &g->shard_ovf, &g->masks, &g->fresh_count, &g->cset})
      b->release(true);
    for (auto& r : g->prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (cudaEvent_t e : g->event_pool) cudaEventDestroy(e);
    if (g->ev_recon) cudaEventDestroy(g->ev_recon);
    for (int i = 0; i < 2; ++i) {
      if (g->ev_copy[i]) cudaEventDestroy(g->ev_copy[i]);
      if (g->ev_used[i]) cudaEventDestroy(g->ev_used[i]);
    }
    if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
    if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
  }
  delete g;
  return SSPD_OK;
}

sspd_status sspd_grid_clone(const sspd_grid* src_c, int device, sspd_grid** out) {
  if (sspd_status w = whole_only(src_c, "clone")) return w;
  auto* src = const_cast<sspd_grid*>(src_c);
  if (sspd_status w = wide_only(src, "Rsea copy")) return w;
  std::lock_guard<std::mutex> lk(src->mu);
  DeviceGuard dg(src->device);
  sspd_status s = commit_locked(src);
  if (s) return s;
  const int dev = device < 0 ? src->device : device;
  s = sspd_grid_create(dev, src->q, src->r, src->delta, src->seed, src->eta, out);
  if (s) return s;
  sspd_grid* g = *out;
  CU(cudaStreamSynchronize(src->stream));
  {
    DeviceGuard dg2(dev);
    CU(cudaMemcpyPeerAsync(g->stamps, dev, src->stamps, src->device, src->geo.n_rec * 4, g->stream));
    g->now = src->now;
    g->pristine = src->pristine;
    if (src->K) {
      g->K = src->K;
      CU(cache_alloc((void**)&g->hist, (size_t)g->K * g->geo.ncells * 4));
      if (src->hist_valid) {
        CU(cudaMemcpyPeerAsync(g->hist, dev, src->hist, src->device, (size_t)g->K * g->geo.ncells * 4,
                               g->stream));
        g->hist_valid = true;
      }
    }
    CU(cudaStreamSynchronize(g->stream));
  }
  return SSPD_OK;
}

sspd_status sspd_grid_info(const sspd_grid* g, uint64_t* recorders, int* device, uint32_t* now) {
  if (recorders) *recorders = g->geo.n_rec;
  if (device) *device = g->device;
  if (now) *now = g->now;
  return SSPD_OK;
}

sspd_status sspd_grid_set_stream(sspd_grid* g, void* cuda_stream) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  CU(cudaStreamSynchronize(g->stream));
  if (g->own_stream) cudaStreamDestroy(g->stream);
  if (cuda_stream) {
    g->stream = static_cast<cudaStream_t>(cuda_stream);
    g->own_stream = false;
  } else {
    CU(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->own_stream = true;
  }
  return SSPD_OK;
}

sspd_status sspd_grid_stream(const sspd_grid* g, void** cuda_stream) {
  *cuda_stream = g->stream;
  return SSPD_OK;
}

sspd_status sspd_grid_synchronize(sspd_grid* g) {
  DeviceGuard dg(g->device);
  CU(cudaStreamSynchronize(g->stream));
  return SSPD_OK;
}

namespace {
sspd_status scan_locked(sspd_grid* g, const uint32_t* pairs, uint64_t n, int pairs_on_device, int stride);
}

sspd_status sspd_scan(sspd_grid* g, const uint32_t* pairs, uint64_t n, int pairs_on_device) {
  if (n == 0) return SSPD_OK;
  if (!pairs) return fail(SSPD_INVALID_ARGUMENT, "scan_batch: null pairs");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  return scan_locked(g, pairs, n, pairs_on_device, 2);
}

sspd_status sspd_scan_records(sspd_grid* g, const uint32_t* records, uint64_t n, int on_device) {
  if (n == 0) return SSPD_OK;
  if (!records) return fail(SSPD_INVALID_ARGUMENT, "scan_records: null records");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (on_device) {  // to pairs on the device, then the pair path
    if (g->rec_pairs.ensure(n * 8) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
    records_to_pairs_kernel<<<grid_blocks(g, n, 256, 8), 256, 0, g->stream>>>(records, n, g->rec_pairs.as<uint2>());
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return scan_locked(g, g->rec_pairs.as<uint32_t>(), n, 1, 2);
  }
  return scan_locked(g, records, n, 0, 3);
}

namespace {
// stride: u32 words per input item -- 2 for (cip, oip) pairs, 3 for
// (ts, cip, oip) trace records (host input only; converted per chunk).
sspd_status scan_locked(sspd_grid* g, const uint32_t* pairs, uint64_t n, int pairs_on_device, int stride) {
  if (g->partial && !g->shard)
    return fail(SSPD_INVALID_ARGUMENT, "scan: a sharded router's partial grid scans through the shard exchange "
                                       "(sspd_set_shard / sspd_set_shard_relay first)");
  g->pristine = false;
  const bool pow2 = (g->eta & (g->eta - 1)) == 0 && g->eta <= (1u << 31);
  // auto: pairs streamed from the host are PCIe-bound, so stamp them in place
  // while the copies run (nothing left to fold after the last chunk);
  // device-resident pairs use the deferred bitmap, which is faster in HBM.
  // auto: never leave deferred work after the last (PCIe) chunk of a host
  // scan; use the pair set once the grid is far beyond L2.
  int mode = g->scan_mode;
  // Measured (profiles/r01_ab_*.txt): with the touched bitmap L2-sized (C1)
  // direct stamping is fastest for host and device pairs alike (0.42 vs 0.46
  // ms/slot bitmap+commit); beyond L2 (C2) the pair set wins (3.9 vs 11.9).
  // Binning by pair-set region first (mode 3) makes the probes L2 hits but
  // measured slower overall (2.2 + 3.6 ms): the random stamp atomics dominate.
  if (mode < 0) mode = g->n_words * 4 > (48ull << 20) ? 2 : 1;
  if (g->width != 32) mode = mode == 0 ? 1 : (mode == 3 ? 2 : mode);  // narrow: direct or dedup
  if ((g->export_pairs || g->shard) && mode < 2) mode = 2;  // only the pair set knows which pairs are new
  // binning pays for itself on large device batches (8-byte aligned pairs)
  const bool use_bins = mode == 3 && pairs_on_device && n >= (4ull << 20) && n < (1ull << 31) &&
                      (reinterpret_cast<uintptr_t>(pairs) & 7u) == 0;
  if (mode == 3) mode = 2;
  const bool direct = mode == 1;
  const bool dedup = mode == 2;
  const bool hist = (direct || dedup) && g->K && g->hist_valid;
  const bool bits = (direct || dedup) && g->record_touched;
  if (g->export_pairs) {
    // new pairs <= pairs scanned this slot, plus each launch's padding of
    // its warps' last list blocks (kernels.cuh list_pad): grow the list,
    // keeping its prefix
    const uint64_t launches = pairs_on_device ? 1 : (n + (4ull << 20) - 1) / (256ull << 10);
    g->list_pad_slots += launches * (uint64_t)sm_count(g->device) * SSPD_SCAN_BLOCKS_PER_SM * 8 * kListBlock;
    const uint64_t need = (g->scanned_in_slot + n + g->list_pad_slots) * 8;
    if (g->newpairs.bytes < need) {
      DevBuf bigger;
      if (bigger.ensure(std::max<uint64_t>(need, g->newpairs.bytes * 2)) != cudaSuccess)
        return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (pair list)");
      if (g->newpairs.p) CU(cudaMemcpyAsync(bigger.p, g->newpairs.p, g->newpairs.bytes, cudaMemcpyDeviceToDevice,
                                            g->stream));
      CU(cudaStreamSynchronize(g->stream));
      g->newpairs.release();
      g->newpairs = bigger;
      bigger.p = nullptr;
    }
    if (!g->newpairs_count.p) {
      if (g->newpairs_count.ensure(8) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
      CU(cudaMemsetAsync(g->newpairs_count.p, 0, 8, g->stream));
    }
  }
  g->scanned_in_slot += n;
  if (!g->shard && g->width == 32 && (bits || (!direct && !dedup)))
    if (sspd_status ts = ensure_touched_locked(g)) return ts;
  // the pipelined dedup path, and within it the compact key set (eta <= 2^16)
  const bool pipe = dedup && !g->shard && !g->export_pairs && hist && !bits && g->width == 32 && g->geo.r <= 8 &&
                    (g->dedup_pipe == 0 || g->dedup_pipe == 1);
  const bool cset = pipe && g->use_cset && g->geo.eta <= 65536u;
  // narrow grids' dedup scan: the same pipelined key-set kernel on bf16 / byte codes
  const bool ncset = dedup && (g->width == 16 || (g->width == 8 && g->cset8)) && !g->shard && !g->export_pairs && g->K && g->geo.r <= 8 &&
                     g->use_cset && g->geo.eta <= 65536u;
  if (cset || ncset) {
    if (sspd_status cs = ensure_cset_locked(g)) return cs;
  } else if (dedup || g->shard) {
    sspd_status ps = ensure_pairset_locked(g);
    if (ps) return ps;
  }
  auto launch = [&](const uint32_t* dp, uint64_t cnt) {
    const unsigned blocks = grid_blocks(g, (cnt + 3) / 4, 256, SSPD_SCAN_BLOCKS_PER_SM);
    Prof p(g, "scan", cnt);
    if (g->shard) {  // own pairs of a sharded router: stamp owned cells, push to the other owners
      auto* tb = g->pairset.as<unsigned long long>();
      const bool hs = g->K && g->hist_valid;
#define SSPD_SHARD(H1, HI, MODE)                                                                                 \
  scan_shard_kernel<H1, HI, MODE><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb, g->pairset_mask, \
                                                                 g->stamps, g->now, g->hist, g->K, g->shard_args)
      if (g->relay) {  // hop 1: new pairs to their pair owners, nothing stamped yet
        if (pow2) SSPD_SHARD(0, 0, kShardToPairOwner);
        else SSPD_SHARD(1, 0, kShardToPairOwner);
      } else if (pow2 && hs) SSPD_SHARD(0, 1, kShardOwn);
      else if (pow2) SSPD_SHARD(0, 0, kShardOwn);
      else if (hs) SSPD_SHARD(1, 1, kShardOwn);
      else SSPD_SHARD(1, 0, kShardOwn);
#undef SSPD_SHARD
      g->pairset_dirty = true;
      return;
    }
    if (ncset) {
      const NarrowCodes nc{g->code_now(), g->code_lo};
      const unsigned pblocks = grid_blocks(g, (cnt + 3) / 4, 256, SSPD_PIPE_MINB);
      auto* ct = g->cset.as<uint32_t>();
      auto* fc = g->fresh_count.as<unsigned long long>();
#define SSPD_CSETN(T, H1, R)                                                                                     \
  scan_cset_kernel<H1, 1, R, SSPD_CSET_BW, T><<<pblocks, 256, 0, g->stream>>>(                                   \
      dp, cnt, g->d_tabs, g->geo, ct, g->cset_lg, static_cast<T*>(g->codes), g->now, g->hist, g->K, fc, 0u, 31u, nc)
      const bool r5 = g->geo.r == 5;
      if (g->width == 8) {
        if (pow2 && r5) SSPD_CSETN(uint8_t, 0, 5);
        else if (pow2) SSPD_CSETN(uint8_t, 0, 0);
        else if (r5) SSPD_CSETN(uint8_t, 1, 5);
        else SSPD_CSETN(uint8_t, 1, 0);
      } else {
        if (pow2 && r5) SSPD_CSETN(uint16_t, 0, 5);
        else if (pow2) SSPD_CSETN(uint16_t, 0, 0);
        else if (r5) SSPD_CSETN(uint16_t, 1, 5);
        else SSPD_CSETN(uint16_t, 1, 0);
      }
#undef SSPD_CSETN
      g->cset_dirty = true;
      return;
    }
    if (g->width != 32) {
      auto* tb = g->pairset.as<unsigned long long>();
      const NarrowCodes nc{g->code_now(), g->code_lo};
#define SSPD_NARROW_PL(T, H1, DD)                                                                    \
  scan_narrow_kernel<T, H1, DD, 1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb, g->pairset_mask, \
                                                                  static_cast<T*>(g->codes), g->now, nc, g->hist, g->K)
#define SSPD_NARROW(T, H1, DD)                                                                       \
  scan_narrow_kernel<T, H1, DD><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb, g->pairset_mask, \
                                                               static_cast<T*>(g->codes), g->now, nc,            \
                                                               g->hist, g->K)
      if (g->width == 8) {
        if (pow2 && dedup) SSPD_NARROW(uint8_t, 0, 1);
        else if (pow2) SSPD_NARROW(uint8_t, 0, 0);
        else if (dedup) SSPD_NARROW(uint8_t, 1, 1);
        else SSPD_NARROW(uint8_t, 1, 0);
      } else if (g->narrow_preload) {
        if (pow2 && dedup) SSPD_NARROW_PL(uint16_t, 0, 1);
        else if (pow2) SSPD_NARROW_PL(uint16_t, 0, 0);
        else if (dedup) SSPD_NARROW_PL(uint16_t, 1, 1);
        else SSPD_NARROW_PL(uint16_t, 1, 0);
      } else {
        if (pow2 && dedup) SSPD_NARROW(uint16_t, 0, 1);
        else if (pow2) SSPD_NARROW(uint16_t, 0, 0);
        else if (dedup) SSPD_NARROW(uint16_t, 1, 1);
        else SSPD_NARROW(uint16_t, 1, 0);
      }
#undef SSPD_NARROW_PL
#undef SSPD_NARROW
      if (dedup) g->pairset_dirty = true;
      return;
    }
    const int F = g->scan_filter;
#define SSPD_DIRECT(H1, FI, HI, BI)                                                                 \
  scan_direct_kernel<H1, FI, HI, BI><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, g->stamps, \
                                                                    g->now, g->hist, g->K, g->touched)
    if (dedup) {
      auto* tb = g->pairset.as<unsigned long long>();
      auto* np = g->newpairs.as<uint2>();
      auto* nc = g->newpairs_count.as<unsigned long long>();
#define SSPD_DEDUP(H1, HI, BI, EX)                                                                  \
  scan_dedup_kernel<H1, HI, BI, EX><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb,          \
                                                                   g->pairset_mask, g->stamps, g->now,      \
                                                                   g->hist, g->K, g->touched, np, nc)
      const bool ex = g->export_pairs;
      if (cset) {
        const unsigned pblocks = grid_blocks(g, (cnt + 3) / 4, 256, SSPD_PIPE_MINB);
        auto* ct = g->cset.as<uint32_t>();
        auto* fc = g->fresh_count.as<unsigned long long>();
        // passes over the batch, each probing 1/passes of the set ($SSPD_CSET_PASSES)
        const uint32_t plog = g->cset_pass_log2;
        const uint32_t lgb = g->cset_lg - (SSPD_CSET_BW == 8 ? 3 : SSPD_CSET_BW == 4 ? 2 : 0);
        const uint32_t pshift = plog ? lgb - plog : 31u;
#define SSPD_CSETK(H1, HI, R)                                                                                    \
  for (uint32_t part = 0; part < (1u << plog); ++part)                                                            \
  scan_cset_kernel<H1, HI, R, SSPD_CSET_BW><<<pblocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, ct,         \
                                                                           g->cset_lg, g->stamps, g->now, g->hist, \
                                                                           g->K, fc, part, pshift)
        const bool r5 = g->geo.r == 5, hint = g->cset_hint != 0;
        switch ((pow2 ? 0 : 4) + (hint ? 2 : 0) + (r5 ? 1 : 0)) {
          case 0: SSPD_CSETK(0, 0, 0); break;
          case 1: SSPD_CSETK(0, 0, 5); break;
          case 2: SSPD_CSETK(0, 1, 0); break;
          case 3: SSPD_CSETK(0, 1, 5); break;
          case 4: SSPD_CSETK(1, 0, 0); break;
          case 5: SSPD_CSETK(1, 0, 5); break;
          case 6: SSPD_CSETK(1, 1, 0); break;
          default: SSPD_CSETK(1, 1, 5); break;
        }
#undef SSPD_CSETK
        g->cset_dirty = true;
      } else if (!ex && hist && !bits && g->geo.r <= 8 && (g->dedup_pipe == 0 || g->dedup_pipe == 1)) {
        // one resident wave of the pipelined kernel (its own occupancy)
        const unsigned pblocks = grid_blocks(g, (cnt + 3) / 4, 256, SSPD_PIPE_MINB);
#define SSPD_PIPE(H1, HI, R)                                                                                 \
  scan_dedup_pipe_kernel<H1, HI, R><<<pblocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb,              \
                                                                   g->pairset_mask, g->stamps, g->now, g->hist,  \
                                                                   g->K, g->fresh_count.as<unsigned long long>())
        const bool r5 = g->geo.r == 5, hint = g->dedup_pipe == 1;
        switch ((pow2 ? 0 : 4) + (hint ? 2 : 0) + (r5 ? 1 : 0)) {
          case 0: SSPD_PIPE(0, 0, 0); break;
          case 1: SSPD_PIPE(0, 0, 5); break;
          case 2: SSPD_PIPE(0, 1, 0); break;
          case 3: SSPD_PIPE(0, 1, 5); break;
          case 4: SSPD_PIPE(1, 0, 0); break;
          case 5: SSPD_PIPE(1, 0, 5); break;
          case 6: SSPD_PIPE(1, 1, 0); break;
          default: SSPD_PIPE(1, 1, 5); break;
        }
#undef SSPD_PIPE
      } else if (ex && g->push.world > 1) {
        if (pow2 && hist)
          scan_dedup_kernel<0, 1, 0, 1, 1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb,
                                                                          g->pairset_mask, g->stamps, g->now,
                                                                          g->hist, g->K, g->touched, np, nc, g->push);
        else if (pow2)
          scan_dedup_kernel<0, 0, 0, 1, 1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb,
                                                                          g->pairset_mask, g->stamps, g->now,
                                                                          g->hist, g->K, g->touched, np, nc, g->push);
        else if (hist)
          scan_dedup_kernel<1, 1, 0, 1, 1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb,
                                                                          g->pairset_mask, g->stamps, g->now,
                                                                          g->hist, g->K, g->touched, np, nc, g->push);
        else
          scan_dedup_kernel<1, 0, 0, 1, 1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, tb,
                                                                          g->pairset_mask, g->stamps, g->now,
                                                                          g->hist, g->K, g->touched, np, nc, g->push);
      } else if (pow2 && ex && hist) SSPD_DEDUP(0, 1, 0, 1);
      else if (pow2 && ex) SSPD_DEDUP(0, 0, 0, 1);
      else if (ex && hist) SSPD_DEDUP(1, 1, 0, 1);
      else if (ex) SSPD_DEDUP(1, 0, 0, 1);
      else if (pow2 && hist && bits) SSPD_DEDUP(0, 1, 1, 0);
      else if (pow2 && hist) SSPD_DEDUP(0, 1, 0, 0);
      else if (pow2 && bits) SSPD_DEDUP(0, 0, 1, 0);
      else if (pow2) SSPD_DEDUP(0, 0, 0, 0);
      else if (hist && bits) SSPD_DEDUP(1, 1, 1, 0);
      else if (hist) SSPD_DEDUP(1, 1, 0, 0);
      else if (bits) SSPD_DEDUP(1, 0, 1, 0);
      else SSPD_DEDUP(1, 0, 0, 0);
#undef SSPD_DEDUP
      g->pairset_dirty = true;
    } else if (!direct) {
      if (pow2 && F) scan_bitmap_kernel<0, 1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, g->touched);
      else if (pow2) scan_bitmap_kernel<0, 0><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, g->touched);
      else if (F) scan_bitmap_kernel<1, 1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, g->touched);
      else scan_bitmap_kernel<1, 0><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, g->touched);
    } else if (pow2) {
      if (F && hist && bits) SSPD_DIRECT(0, 1, 1, 1);
      else if (F && hist) SSPD_DIRECT(0, 1, 1, 0);
      else if (F && bits) SSPD_DIRECT(0, 1, 0, 1);
      else if (F) SSPD_DIRECT(0, 1, 0, 0);
      else if (hist && bits) SSPD_DIRECT(0, 0, 1, 1);
      else if (hist) SSPD_DIRECT(0, 0, 1, 0);
      else if (bits) SSPD_DIRECT(0, 0, 0, 1);
      else SSPD_DIRECT(0, 0, 0, 0);
    } else {
      if (hist && bits) SSPD_DIRECT(1, 1, 1, 1);
      else if (hist) SSPD_DIRECT(1, 1, 1, 0);
      else if (bits) SSPD_DIRECT(1, 1, 0, 1);
      else SSPD_DIRECT(1, 1, 0, 0);
    }
#undef SSPD_DIRECT
  };
  // Direct scans stamp in place; only recorded bits (multi-router) or a
  // stale window ring leave work for the commit.
  if (!(direct || dedup) || (bits && !g->export_pairs)) g->pending = true;
  if (pairs_on_device && use_bins) {
    // partition by pair-set region, then one dedup pass in region order
    const unsigned G = (unsigned)sm_count(g->device) * 8;
    const uint64_t chunk = (n + G - 1) / G;
    if (g->bin_counts.ensure((size_t)kPairBins * G * 4) != cudaSuccess || g->binned.ensure(n * 8) != cudaSuccess)
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (binning)");
    uint32_t* counts = g->bin_counts.as<uint32_t>();
    {
      Prof p(g, "bin", n);
      bin_count_kernel<<<G, 256, 0, g->stream>>>(pairs, n, chunk, counts);
      bin_offsets_kernel<<<1, 1024, 0, g->stream>>>(counts, kPairBins * G);
      bin_scatter_kernel<<<G, 256, 0, g->stream>>>(pairs, n, chunk, counts, g->binned.as<uint2>());
    }
    g_launches.fetch_add(2, std::memory_order_relaxed);
    launch(g->binned.as<uint32_t>(), n);
    return check_launch();
  }
  if (pairs_on_device) {
    launch(pairs, n);
    return check_launch();
  }
  // Host pairs: double-buffered chunks; the copy stream fills one staging
  // buffer while the scan consumes the other.
  // Pairs per chunk: at most 4M (32 MiB: small first-copy latency), and at
  // least 4 chunks down to 256K pairs, so the copy of a chunk overlaps the
  // scan of the one before even for a C1-sized (1M-pair) batch.
  const uint64_t chunk_pairs = std::min<uint64_t>(
      n, std::min<uint64_t>(4ull << 20, std::max<uint64_t>(256ull << 10, (n + 3) / 4)));
  // Pageable sources: the driver's own staging copies them at ~11 GB/s
  // (profiles/r01_bench_api.md); instead the host threads pack each chunk
  // into a pinned buffer -- as 8-byte pairs, so records lose their ts on the
  // way -- and DMA copies that at full PCIe speed, overlapping the packing
  // of the next chunk.
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, pairs) != cudaSuccess) cudaGetLastError();
  const bool pinned = attr.type == cudaMemoryTypeHost;
  const bool pack = !pinned && n >= 4096;  // tiny batches: the driver's staged copy is as fast
  const int dstride = pack ? 2 : stride;  // u32 words per item as copied to the device
  for (int i = 0; i < 2; ++i)
    if (g->stage[i].ensure(chunk_pairs * 4 * dstride) != cudaSuccess ||
        (dstride == 3 && g->stage_pairs[i].ensure(chunk_pairs * 8) != cudaSuccess))
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (scan staging)");
  if (pack && g->host_stage_bytes < chunk_pairs * 8) {
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventSynchronize(g->ev_hcopy[i]));
      PinnedCache::get().free(g->host_stage[i]);
      g->host_stage[i] = nullptr;
    }
    g->host_stage_bytes = 0;
    for (int i = 0; i < 2; ++i)
      if (PinnedCache::get().alloc(&g->host_stage[i], chunk_pairs * 8) != cudaSuccess)
        return fail(SSPD_CUDA_ERROR, "CUDA error: pinned scan staging");
    g->host_stage_bytes = chunk_pairs * 8;
  }
  // Balanced chunks; the staging buffer alternates across calls too, so a
  // call's first copy overlaps the previous call's last scan (ev_used[b]:
  // the last scan that read stage[b] -- the copy stream must not overwrite
  // staging still being read).
  const uint64_t n_chunks = (n + chunk_pairs - 1) / chunk_pairs;
  uint64_t done = 0;
  int& buf = g->stage_next;
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const uint64_t cnt = n * (c + 1) / n_chunks - done;
    const uint32_t* src = pairs + (uint64_t)stride * done;
    if (pack) {
      CU(cudaEventSynchronize(g->ev_hcopy[buf]));  // the last DMA out of this pinned buffer is done
      auto* dst = static_cast<uint2*>(g->host_stage[buf]);
      // ~64K items (0.5-0.8 MB) per thread
      const unsigned threads = static_cast<unsigned>(std::min<uint64_t>(16, std::max<uint64_t>(1, cnt >> 16)));
      HostPool::get().run(threads, [&](unsigned t, unsigned T) {
        const uint64_t a = cnt * t / T, b = cnt * (t + 1) / T;
        if (stride == 3) {
          for (uint64_t i = a; i < b; ++i) dst[i] = make_uint2(src[3 * i + 1], src[3 * i + 2]);
        } else if (b > a) {
          std::memcpy(dst + a, src + 2 * a, (b - a) * 8);
        }
      });
      src = static_cast<const uint32_t*>(g->host_stage[buf]);
    }
    CU(cudaStreamWaitEvent(g->copy_stream, g->ev_used[buf], 0));
    CU(cudaMemcpyAsync(g->stage[buf].p, src, cnt * 4 * dstride, cudaMemcpyHostToDevice, g->copy_stream));
    g->h2d_bytes += cnt * 4 * dstride;
    CU(cudaEventRecord(g->ev_copy[buf], g->copy_stream));
    if (pack) CU(cudaEventRecord(g->ev_hcopy[buf], g->copy_stream));
    CU(cudaStreamWaitEvent(g->stream, g->ev_copy[buf], 0));
    if (dstride == 3) {
      records_to_pairs_kernel<<<grid_blocks(g, cnt, 256, 8), 256, 0, g->stream>>>(
          g->stage[buf].as<uint32_t>(), cnt, g->stage_pairs[buf].as<uint2>());
      g_launches.fetch_add(1, std::memory_order_relaxed);
      launch(g->stage_pairs[buf].as<uint32_t>(), cnt);
    } else {
      launch(g->stage[buf].as<uint32_t>(), cnt);
    }
    CU(cudaEventRecord(g->ev_used[buf], g->stream));
    done += cnt;
    buf ^= 1;
  }
  // Pageable sources are consumed by the time the call returns (packed, or
  // staged by the driver inside cudaMemcpyAsync); pinned ones are read by
  // DMA later, and the caller may reuse its buffer on return (scan_batch
  // semantics), so wait for those copies.
  if (pinned) CU(cudaStreamSynchronize(g->copy_stream));
  return check_launch();
}
}  // namespace

sspd_status sspd_commit(sspd_grid* g) {
  if (sspd_status w = whole_only(g, "commit")) return w;
  if (sspd_status w = wide_only(g, "commit")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  g->pristine = false;
  if (!g->touched) return SSPD_OK;  // no bitmap yet: nothing recorded or merged into one
  g->pending = true;  // the caller may have OR-merged remote touches in
  return commit_locked(g);
}

sspd_status sspd_advance(sspd_grid* g, uint32_t slots) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (g->cset_dirty) {
    s = cset_slot_end_locked(g);
    if (s) return s;
  }
  s = pairset_reset_locked(g);  // the pair set only deduplicates within a slot
  if (s) return s;
  if (g->newpairs_count.p) CU(cudaMemsetAsync(g->newpairs_count.p, 0, 8, g->stream));
  if (g->shard) CU(cudaMemsetAsync(g->shard_sent.p, 0, 64 * 8, g->stream));
  if (g->relayset_dirty) {
    CU(cudaMemsetAsync(g->relayset.p, 0xff, g->relayset.bytes, g->stream));
    g->relayset_dirty = false;
  }
  g->scanned_in_slot = 0;
  g->list_pad_slots = 0;
  for (uint32_t i = 0; i < slots; ++i) {
    if (g->now >= 0x7fffffffu) return fail(SSPD_OUT_OF_RANGE, "advance_slot: slice counter exhausted");
    ++g->now;
    if (g->K && g->hist_valid) {
      // the ring entry of the slot leaving the window becomes `now`'s
      CU(cudaMemsetAsync(g->hist + (uint64_t)(g->now % g->K) * g->geo.ncells, 0, (size_t)g->geo.ncells * 4,
                         g->stream));
    }
    if (g->width != 32 && g->code_now() > g->code_hi) {
      // epoch end: drop codes older than the window, move the rest down so
      // that code(now) = lo + K - 1 (ages unchanged)
      const uint32_t cn = g->code_now(), shift = cn - (g->code_lo + g->K - 1);
      const unsigned blocks = grid_blocks(g, g->geo.n_rec / 16 + 1, 256, 8);
      Prof p(g, "rebase", g->geo.n_rec);
      if (g->width == 8)
        narrow_rebase_kernel<uint8_t><<<blocks, 256, 0, g->stream>>>(static_cast<uint8_t*>(g->codes),
                                                                     g->geo.n_rec, cn, g->code_lo, g->K, shift);
      else
        narrow_rebase_kernel<uint16_t><<<blocks, 256, 0, g->stream>>>(static_cast<uint16_t*>(g->codes),
                                                                      g->geo.n_rec, cn, g->code_lo, g->K, shift);
      g->epoch0 = g->now - (g->K - 1);
      s = check_launch();
      if (s) return s;
    }
  }
  return SSPD_OK;
}

sspd_status sspd_get_distances(sspd_grid* g, uint16_t* host_out, uint64_t offset, uint64_t count) {
  if (sspd_status w = wide_only(g, "cells")) return w;
  if (offset > g->geo.n_rec || count > g->geo.n_rec - offset)
    return fail(SSPD_OUT_OF_RANGE, "cells: range out of bounds");
  if (g->partial && count &&
      (offset < (uint64_t)g->geo.own_lo * g->eta || offset + count > (uint64_t)g->geo.own_hi * g->eta))
    return whole_only(g, "cells");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  const uint64_t chunk = 32ull << 20;
  if (g->misc.ensure(std::min(chunk, std::max<uint64_t>(count, 1)) * 2) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (cells)");
  for (uint64_t done = 0; done < count;) {
    const uint64_t cnt = std::min(chunk, count - done);
    {
      Prof p(g, "to_distance", cnt);
      stamps_to_dist_kernel<<<grid_blocks(g, cnt, 256, 8), 256, 0, g->stream>>>(
          g->stamps + offset + done, cnt, g->now, g->misc.as<uint16_t>());
    }
    CU(cudaMemcpyAsync(host_out + done, g->misc.p, cnt * 2, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (cnt * 2);
    CU(cudaStreamSynchronize(g->stream));
    done += cnt;
  }
  return check_launch();
}

sspd_status sspd_put_distances(sspd_grid* g, const uint16_t* host_in, uint64_t offset, uint64_t count) {
  if (sspd_status w = wide_only(g, "cells")) return w;
  if (offset > g->geo.n_rec || count > g->geo.n_rec - offset)
    return fail(SSPD_OUT_OF_RANGE, "cells: range out of bounds");
  if (g->partial && count &&
      (offset < (uint64_t)g->geo.own_lo * g->eta || offset + count > (uint64_t)g->geo.own_hi * g->eta))
    return whole_only(g, "cells");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  s = pairset_reset_locked(g);
  if (s) return s;
  const uint64_t chunk = 32ull << 20;
  if (g->misc.ensure(std::min(chunk, std::max<uint64_t>(count, 1)) * 2) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (cells)");
  for (uint64_t done = 0; done < count;) {
    const uint64_t cnt = std::min(chunk, count - done);
    CU(cudaMemcpyAsync(g->misc.p, host_in + done, cnt * 2, cudaMemcpyHostToDevice, g->stream));
  g->h2d_bytes += (cnt * 2);
    {
      Prof p(g, "from_distance", cnt);
      dist_to_stamps_kernel<<<grid_blocks(g, cnt, 256, 8), 256, 0, g->stream>>>(
          g->misc.as<uint16_t>(), cnt, g->now, g->stamps + offset + done);
    }
    CU(cudaStreamSynchronize(g->stream));
    done += cnt;
  }
  g->hist_valid = false;
  g->pristine = false;
  return check_launch();
}

sspd_status sspd_active_counts(sspd_grid* g, uint32_t k, uint32_t* host_out) {
  if (sspd_status w = whole_only(g, "active_counts")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = counts_locked(g, k);
  if (s) return s;
  CU(cudaMemcpyAsync(host_out, g->counts.p, (size_t)g->geo.ncells * 4, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += ((size_t)g->geo.ncells * 4);
  CU(cudaStreamSynchronize(g->stream));
  return SSPD_OK;
}

sspd_status sspd_hot_sets(sspd_grid* g, uint32_t k, uint64_t cutoff, uint32_t* cols_out, uint32_t* row_counts) {
  if (sspd_status w = whole_only(g, "hot_sets")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  std::vector<uint32_t> rc;
  sspd_status s = hot_locked(g, k, cutoff, &rc, nullptr);
  if (s) return s;
  const uint32_t ncol = 1u << g->q;
  uint64_t pos = 0;
  for (uint32_t row = 0; row < g->r; ++row) {
    row_counts[row] = rc[row];
    if (rc[row])
      CU(cudaMemcpyAsync(cols_out + pos, g->hot_cols.as<uint32_t>() + (uint64_t)row * ncol, rc[row] * 4,
                         cudaMemcpyDeviceToHost, g->stream));
    pos += rc[row];
  }
  g->d2h_bytes += pos * 4;
  CU(cudaStreamSynchronize(g->stream));
  return SSPD_OK;
}

sspd_status sspd_finalize(sspd_grid* g, const uint32_t* tuples, uint64_t n, uint32_t k, uint64_t cutoff,
                          uint8_t* accepted, uint32_t* cips, uint32_t* r_ks) {
  if (sspd_status w = whole_only(g, "finalize_candidate")) return w;
  if (g->r > 64) return fail(SSPD_INVALID_ARGUMENT, "finalize_candidate: r > 64 unsupported");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (sspd_status s = no_pending(g, "finalize_candidate")) return s;
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (n == 0) return SSPD_OK;
  if (g->tupA.ensure(n * g->r * 4) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
  s = ensure_surv(g, n);
  if (s) return s;
  CU(cudaMemcpyAsync(g->tupA.p, tuples, n * g->r * 4, cudaMemcpyHostToDevice, g->stream));
  g->h2d_bytes += n * g->r * 4;
  std::memset(g->meta_host, 0, sizeof(ReconMeta));
  g->meta_host->level[g->r - 1] = n;
  CU(cudaMemcpyAsync(g->meta.p, g->meta_host, sizeof(ReconMeta), cudaMemcpyHostToDevice, g->stream));
  s = queue_finalize(g, g->tupA.as<uint32_t>(), n, k);
  if (s) return s;
  CU(cudaMemcpyAsync(g->meta_host, g->meta.p, sizeof(ReconMeta), cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  const uint64_t ns = g->meta_host->surv;
  std::vector<uint32_t> buf(ns * 3 + 1);
  const uint32_t* s_idx = g->surv.as<uint32_t>();
  if (ns) {
    CU(cudaMemcpyAsync(buf.data(), s_idx, ns * 4, cudaMemcpyDeviceToHost, g->stream));
    CU(cudaMemcpyAsync(buf.data() + ns, s_idx + n, ns * 4, cudaMemcpyDeviceToHost, g->stream));
    CU(cudaMemcpyAsync(buf.data() + 2 * ns, s_idx + 2 * n, ns * 4, cudaMemcpyDeviceToHost, g->stream));
    CU(cudaStreamSynchronize(g->stream));
  }
  g->d2h_bytes += sizeof(ReconMeta) + ns * 12;
  std::memset(accepted, 0, n);
  for (uint64_t i = 0; i < ns; ++i) {
    const uint32_t t = buf[i], rk = buf[2 * ns + i];
    if (rk >= cutoff) {
      accepted[t] = 1;
      cips[t] = buf[ns + i];
      r_ks[t] = rk;
    }
  }
  return SSPD_OK;
}

}  // extern "C"

namespace {

enum class RecStep { kSurvivors, kEmptyRow, kRetry };

// One reconstruction attempt up to the survivors of finalize_check: hot
// compaction (from the stamps, or from OR-merged hot bits when from_words),
// the joins of levels 2..r-1, finalize_check and -- unless sharded --
// finalize_count, all queued; then one synchronisation reads the row and
// level counts (plus a prefix of the survivors).  Overflow is decided level
// by level, as the reference does (rsea.cpp:206-216); a level whose count
// exceeds the buffer but not the cap asks for a re-run with larger buffers.
sspd_status recon_queue(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap, bool from_words, bool count_rk,
                        uint64_t* C_out) {
  const uint32_t ncol = 1u << g->q;
  const uint32_t wpk = words_per_key(g);
  const uint64_t t_stride = (uint64_t)wpk << (g->q - g->delta);
  ReconMeta* meta = g->meta.as<ReconMeta>();
  ReconMeta* mh = g->meta_host;
  if (g->cap_alloc == 0) g->cap_alloc = std::min<uint64_t>(cap, 1u << 20);
  const uint64_t C = std::max<uint64_t>(g->cap_alloc, 1);
  *C_out = C;
  if (g->tupA.ensure(C * g->r * 4) != cudaSuccess || g->tupB.ensure(C * g->r * 4) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (candidate buffer)");
  sspd_status s = ensure_surv(g, C);
  if (s) return s;
  // One event pair around the chain when profiling (events between its
  // kernels would break the programmatic dependent launches).
  Prof chain(g, "reconstruct", C, false);
  ++g->prof_suspend;
  struct Resume {
    sspd_grid* g;
    ~Resume() { --g->prof_suspend; }
  } resume{g};
  // hot_mark zeroes the bookkeeping (meta) before anything reads it
  s = hot_locked(g, k, cutoff, nullptr, meta->rowcnt, from_words, reinterpret_cast<unsigned long long*>(meta),
                 sizeof(ReconMeta) / 8);
  if (s) return s;
  const uint32_t* cols = g->hot_cols.as<uint32_t>();
  const uint32_t* T = g->hotT.as<uint32_t>();
  // level sizes live on the device; a modest persistent grid keeps the
  // (usually tiny) joins cheap to launch and still strides large levels
  const unsigned blocks = (unsigned)sm_count(g->device) * 2;
  s = launch_pdl(g, level2_kernel, blocks, 256, cols, ncol, T + 2 * t_stride, wpk, g->geo, g->tupA.as<uint32_t>(), C,
                 meta);
  if (s) return s;
  DevBuf* rd = &g->tupA;
  DevBuf* wr = &g->tupB;
  for (uint32_t row = 3; row < g->r; ++row) {
    s = launch_pdl(g, level_ext_kernel, blocks, 256, (const uint32_t*)rd->as<uint32_t>(), C, row,
                   T + (uint64_t)row * t_stride, wpk, g->geo, wr->as<uint32_t>(), C, meta);
    if (s) return s;
    std::swap(rd, wr);
  }
  g->last_tuples = rd;
  uint32_t* s_idx = g->surv.as<uint32_t>();
  if (count_rk) {
    s = queue_finalize(g, rd->as<uint32_t>(), C, k);
  } else {
    s = launch_pdl(g, finalize_check_kernel, grid_blocks(g, C, 256, 2), 256, (const uint32_t*)rd->as<uint32_t>(), C,
                   (const HashTabs*)g->d_tabs, g->geo, meta, s_idx, s_idx + C, (uint32_t*)nullptr);
  }
  if (s) return s;
  // Survivors are few (true super points plus hash-consistent impostors):
  // copy a fixed prefix in the same batch.
  uint32_t* hbuf = static_cast<uint32_t*>(g->pinned_small);  // 4 KB: 2 x 512 entries
  const uint64_t pre_small = std::min<uint64_t>(C, 512);
  CU(cudaMemcpyAsync(mh, meta, sizeof(ReconMeta), cudaMemcpyDeviceToHost, g->stream));
  if (count_rk) {
    CU(cudaMemcpyAsync(hbuf, s_idx + C, pre_small * 4, cudaMemcpyDeviceToHost, g->stream));
    CU(cudaMemcpyAsync(hbuf + 512, s_idx + 2 * C, pre_small * 4, cudaMemcpyDeviceToHost, g->stream));
    g->d2h_bytes += pre_small * 8;
  }
  g->d2h_bytes += sizeof(ReconMeta);
  return SSPD_OK;
}

// After the queued attempt has completed: the row and level counts decide.
sspd_status recon_decide(sspd_grid* g, uint64_t cap, uint64_t C, RecStep* step, uint32_t* ovf_level,
                         uint64_t* ovf_count) {
  const ReconMeta* mh = g->meta_host;
  *step = RecStep::kSurvivors;
  for (uint32_t row = 0; row < g->r; ++row)
    if (mh->rowcnt[row] == 0) {  // rsea.cpp:173-174
      *step = RecStep::kEmptyRow;
      return SSPD_OK;
    }
  for (uint32_t lvl = 2; lvl < g->r; ++lvl) {
    const uint64_t cnt = mh->level[lvl];
    if (cnt > cap) {
      *ovf_level = lvl;
      *ovf_count = cnt;
      return fail(SSPD_CANDIDATE_OVERFLOW, "candidate buffer cap exceeded at level " + std::to_string(lvl) + ": " +
                                               std::to_string(cnt) + " tuples, cap " + std::to_string(cap));
    }
    if (cnt > C) {
      g->cap_alloc = cnt;
      *step = RecStep::kRetry;
      return SSPD_OK;
    }
  }
  return SSPD_OK;
}

sspd_status recon_attempt(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap, bool from_words, bool count_rk,
                          uint64_t* C_out, RecStep* step, uint32_t* ovf_level, uint64_t* ovf_count) {
  sspd_status s = recon_queue(g, k, cutoff, cap, from_words, count_rk, C_out);
  if (s) return s;
  CU(cudaStreamSynchronize(g->stream));
  return recon_decide(g, cap, *C_out, step, ovf_level, ovf_count);
}

// The survivors' (cip, R_k) of a completed count_rk attempt: the pinned
// prefix, or a read-back of all of them (on the copy stream, after `after`).
sspd_status survivors(sspd_grid* g, uint64_t C, cudaEvent_t after, std::vector<uint32_t>* cip,
                      std::vector<uint32_t>* rk) {
  const uint64_t ns = g->meta_host->surv;
  const uint32_t* hbuf = static_cast<const uint32_t*>(g->pinned_small);
  const uint32_t* s_idx = g->surv.as<uint32_t>();
  cip->resize(ns);
  rk->resize(ns);
  if (ns <= std::min<uint64_t>(C, 512)) {
    std::memcpy(cip->data(), hbuf, ns * 4);
    std::memcpy(rk->data(), hbuf + 512, ns * 4);
    return SSPD_OK;
  }
  cudaStream_t st = after ? g->copy_stream : g->stream;
  if (after) CU(cudaStreamWaitEvent(st, after, 0));
  CU(cudaMemcpyAsync(cip->data(), s_idx + C, ns * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(rk->data(), s_idx + 2 * C, ns * 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  g->d2h_bytes += ns * 8;
  return SSPD_OK;
}


// dedup_report (rsea.cpp:112-122) of the survivors' (cip, R_k): by cip,
// larger estimate kept, sorted by cip; estimates in host double.
void report(const sspd_grid* g, const std::vector<uint32_t>& cip, const std::vector<uint32_t>& rk, uint64_t cutoff,
            sspd_detection* out, uint64_t out_cap, uint64_t* n_out) {
  std::map<uint32_t, uint32_t> best;
  for (size_t i = 0; i < cip.size(); ++i) {
    if (rk[i] < cutoff) continue;
    auto it = best.emplace(cip[i], rk[i]);
    if (!it.second && rk[i] > it.first->second) it.first->second = rk[i];
  }
  *n_out = best.size();
  uint64_t w = 0;
  for (const auto& [c, r_k] : best) {
    if (w < out_cap) out[w] = sspd_detection{c, r_k, estimate(g->eta, r_k)};
    ++w;
  }
}

}  // namespace

extern "C" {

sspd_status sspd_reconstruct(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap, sspd_detection* out,
                             uint64_t out_cap, uint64_t* n_out, uint32_t* ovf_level, uint64_t* ovf_count) {
  *n_out = 0;
  if (sspd_status w = whole_only(g, "reconstruct")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (sspd_status s = no_pending(g, "reconstruct")) return s;
  if (g->r > 64) return fail(SSPD_INVALID_ARGUMENT, "reconstruct: r > 64 unsupported");
  if (g->shard && g->shard_args.world > 1)
    return fail(SSPD_INVALID_ARGUMENT, "reconstruct: a sharded grid reconstructs through the shard calls");
  for (int attempt = 0;; ++attempt) {
    uint64_t C = 0;
    RecStep step;
    sspd_status s = recon_attempt(g, k, cutoff, cap, false, true, &C, &step, ovf_level, ovf_count);
    if (s) return s;
    if (step == RecStep::kEmptyRow) return SSPD_OK;
    if (step == RecStep::kRetry) {
      if (attempt > 8) return fail(SSPD_CUDA_ERROR, "reconstruct: candidate buffer did not converge");
      continue;
    }
    std::vector<uint32_t> cip, rk;
    s = survivors(g, C, nullptr, &cip, &rk);
    if (s) return s;
    report(g, cip, rk, cutoff, out, out_cap, n_out);
    return SSPD_OK;
  }
}

sspd_status sspd_reconstruct_async(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap) {
  if (sspd_status w = whole_only(g, "reconstruct")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (sspd_status s = no_pending(g, "reconstruct_async")) return s;
  if (g->r > 64) return fail(SSPD_INVALID_ARGUMENT, "reconstruct: r > 64 unsupported");
  if (g->shard && g->shard_args.world > 1)
    return fail(SSPD_INVALID_ARGUMENT, "reconstruct: a sharded grid reconstructs through the shard calls");
  if (cap > (1ull << 26)) return fail(SSPD_INVALID_ARGUMENT, "reconstruct_async: cap above 2^26 tuples");
  // buffers for `cap` tuples up front: a level either fits or overflows the
  // cap, so collect never has to re-run anything
  g->cap_alloc = std::max<uint64_t>(g->cap_alloc, std::max<uint64_t>(cap, 1));
  uint64_t C = 0;
  sspd_status s = recon_queue(g, k, cutoff, cap, false, true, &C);
  if (s) return s;
  CU(cudaEventRecord(g->ev_recon, g->stream));
  g->recon_pending = true;
  g->collected_ready = false;
  g->pend_cutoff = cutoff;
  g->pend_cap = cap;
  g->pend_C = C;
  return SSPD_OK;
}

sspd_status sspd_reconstruct_collect(sspd_grid* g, sspd_detection* out, uint64_t out_cap, uint64_t* n_out,
                                     uint32_t* ovf_level, uint64_t* ovf_count) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  *n_out = 0;
  if (!g->recon_pending && !g->collected_ready)
    return fail(SSPD_INVALID_ARGUMENT, "reconstruct_collect: nothing queued");
  if (g->recon_pending) {
    g->recon_pending = false;
    g->collected.clear();
    CU(cudaEventSynchronize(g->ev_recon));
    RecStep step;
    sspd_status s = recon_decide(g, g->pend_cap, g->pend_C, &step, ovf_level, ovf_count);
    if (s) return s;
    if (step == RecStep::kRetry) return fail(SSPD_CUDA_ERROR, "reconstruct_collect: candidate buffer too small");
    if (step == RecStep::kSurvivors) {
      std::vector<uint32_t> cip, rk;
      s = survivors(g, g->pend_C, g->ev_recon, &cip, &rk);
      if (s) return s;
      uint64_t n = 0;
      report(g, cip, rk, g->pend_cutoff, nullptr, 0, &n);
      g->collected.resize(n);
      report(g, cip, rk, g->pend_cutoff, g->collected.data(), n, &n);
    }
    g->collected_ready = true;
  }
  // the reports stay readable (e.g. again with a larger buffer) until the next queue
  *n_out = g->collected.size();
  std::memcpy(out, g->collected.data(), std::min<uint64_t>(out_cap, g->collected.size()) * sizeof(sspd_detection));
  return SSPD_OK;
}

// ---- sharded routers ----

sspd_status sspd_set_shard(sspd_grid* g, void* dev_inbox_ptrs, uint32_t world, uint32_t rank, uint64_t region_cap) {
  if (sspd_status w = wide_only(g, "set_shard")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (g->partial && (world != g->part_world || rank != g->part_rank))
    return fail(SSPD_INVALID_ARGUMENT, "set_shard: this partial grid was created for router " +
                                           std::to_string(g->part_rank) + " of " + std::to_string(g->part_world));
  if (world == 0) {
    g->shard = false;
    return SSPD_OK;
  }
  if (world > 32 || rank >= world || (world > 1 && (!dev_inbox_ptrs || region_cap == 0)))
    return fail(SSPD_INVALID_ARGUMENT, "set_shard: need world <= 32, rank < world, inboxes and region_cap > 0");
  if (g->export_pairs || g->record_touched)
    return fail(SSPD_INVALID_ARGUMENT, "set_shard: turn the other exchange hooks off first");
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (g->shard_sent.ensure(64 * 8) != cudaSuccess || g->shard_ovf.ensure(4) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
  CU(cudaMemsetAsync(g->shard_sent.p, 0, 64 * 8, g->stream));
  CU(cudaMemsetAsync(g->shard_ovf.p, 0, 4, g->stream));
  g->shard_args = ShardArgs{static_cast<uint2* const*>(dev_inbox_ptrs), g->shard_sent.as<unsigned long long>(),
                            world, rank, region_cap};
  g->shard = true;
  g->relay = false;
  return SSPD_OK;
}

sspd_status sspd_set_shard_relay(sspd_grid* g, void* dev_inbox_a, void* dev_inbox_b, uint32_t world, uint32_t rank,
                                 uint64_t region_cap) {
  sspd_status s = sspd_set_shard(g, dev_inbox_a, world, rank, region_cap);
  if (s || world == 0) return s;
  std::lock_guard<std::mutex> lk(g->mu);
  if (world > 1 && !dev_inbox_b) return fail(SSPD_INVALID_ARGUMENT, "set_shard_relay: need both inbox tables");
  g->shard_b = ShardArgs{static_cast<uint2* const*>(dev_inbox_b), g->shard_sent.as<unsigned long long>() + 32, world,
                         rank, region_cap};
  g->relay = true;
  return SSPD_OK;
}

sspd_status sspd_shard_sent(sspd_grid* g, uint64_t** dev_counts) {
  std::lock_guard<std::mutex> lk(g->mu);
  if (!g->shard) return fail(SSPD_INVALID_ARGUMENT, "shard_sent: not a sharded grid");
  *dev_counts = reinterpret_cast<uint64_t*>(g->shard_sent.p);
  return SSPD_OK;
}

namespace {
sspd_status shard_receive_locked(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n, const ShardSegs& segs);
}

sspd_status sspd_shard_receive(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n) {
  if (n == 0) return SSPD_OK;
  std::lock_guard<std::mutex> lk(g->mu);
  return shard_receive_locked(g, dev_pairs, n, ShardSegs{});
}

namespace {
// Device-counted segments (kernels.cuh ShardSegs::dev_counts): launched with
// a grid sized for the regions' capacity; the kernel reads the counts.
ShardSegs dev_segs(sspd_grid* g, uint64_t region_stride, const uint64_t* dev_counts, uint64_t count_stride,
                   uint32_t n_regions, uint32_t skip) {
  ShardSegs segs{};
  segs.stride = region_stride;
  segs.nseg = n_regions;
  segs.skip = skip;
  segs.dev_counts = reinterpret_cast<const unsigned long long*>(dev_counts);
  segs.count_stride = count_stride;
  segs.ovf = g->shard_ovf.as<uint32_t>();
  return segs;
}
}  // namespace

sspd_status sspd_shard_receive_regions_dev(sspd_grid* g, const uint32_t* dev_base, uint64_t region_stride,
                                           const uint64_t* dev_counts, uint64_t count_stride, uint32_t n_regions,
                                           uint32_t skip_region) {
  if (n_regions == 0 || n_regions > 32 || !dev_counts)
    return fail(SSPD_INVALID_ARGUMENT, "shard_receive_regions: 1..32 regions and device counts");
  std::lock_guard<std::mutex> lk(g->mu);
  if (!g->shard) return fail(SSPD_INVALID_ARGUMENT, "shard_receive: not a sharded grid");
  return shard_receive_locked(g, dev_base, region_stride * n_regions,
                              dev_segs(g, region_stride, dev_counts, count_stride, n_regions, skip_region));
}

sspd_status sspd_reduce_words(int device, const uint32_t* const* srcs, uint32_t n_src, uint64_t words, int op,
                              uint32_t* dst, void* cuda_stream) {
  if (n_src == 0 || n_src > 32 || (op != 0 && op != 1) || !dst)
    return fail(SSPD_INVALID_ARGUMENT, "reduce_words: 1..32 sources, op 0 (OR) or 1 (AND)");
  if (words == 0) return SSPD_OK;
  DeviceGuard dg(device);
  ReduceSrcs rs{};
  bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15u) == 0;
  for (uint32_t i = 0; i < n_src; ++i) {
    if (!srcs[i]) return fail(SSPD_INVALID_ARGUMENT, "reduce_words: null source");
    rs.p[i] = srcs[i];
    aligned = aligned && (reinterpret_cast<uintptr_t>(srcs[i]) & 15u) == 0;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const uint64_t items = aligned ? (words + 3) / 4 : words;
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((items + 255) / 256, (uint64_t)sms * 4));
  auto st = static_cast<cudaStream_t>(cuda_stream);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (op) reduce_words_kernel<1><<<blocks, 256, 0, st>>>(rs, n_src, words, dst, aligned ? 1 : 0);
  else reduce_words_kernel<0><<<blocks, 256, 0, st>>>(rs, n_src, words, dst, aligned ? 1 : 0);
  return check_launch();
}

sspd_status sspd_shard_overflow(sspd_grid* g, int* overflowed) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  *overflowed = 0;
  if (!g->shard_ovf.p) return SSPD_OK;
  CU(cudaMemcpyAsync(pinned_scratch(g), g->shard_ovf.p, 4, cudaMemcpyDeviceToHost, g->stream));
  CU(cudaMemsetAsync(g->shard_ovf.p, 0, 4, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  *overflowed = *static_cast<int*>(pinned_scratch(g)) != 0;
  return SSPD_OK;
}

namespace {
sspd_status shard_receive_locked(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n, const ShardSegs& segs) {
  DeviceGuard dg(g->device);
  if (!g->shard) return fail(SSPD_INVALID_ARGUMENT, "shard_receive: not a sharded grid");
  sspd_status s = ensure_pairset_locked(g);
  if (s) return s;
  g->pristine = false;
  g->pairset_dirty = true;
  const bool pow2 = (g->eta & (g->eta - 1)) == 0 && g->eta <= (1u << 31);
  const bool hist = g->K && g->hist_valid;
  const unsigned blocks = grid_blocks(g, (n + 3) / 4, 256, SSPD_SCAN_BLOCKS_PER_SM);
  auto* tb = g->pairset.as<unsigned long long>();
  Prof p(g, "scan", n);
#define SSPD_SHARD(H1, HI, MODE)                                                                             \
  scan_shard_kernel<H1, HI, MODE><<<blocks, 256, 0, g->stream>>>(dev_pairs, n, g->d_tabs, g->geo, tb,          \
                                                                 g->pairset_mask, g->stamps, g->now, g->hist, g->K, \
                                                                 g->shard_args, segs)
  if (g->relay) {  // hop 2: each pair arrives once from its pair owner
    if (pow2 && hist) SSPD_SHARD(0, 1, kShardRecvOnce);
    else if (pow2) SSPD_SHARD(0, 0, kShardRecvOnce);
    else if (hist) SSPD_SHARD(1, 1, kShardRecvOnce);
    else SSPD_SHARD(1, 0, kShardRecvOnce);
  } else if (pow2 && hist) SSPD_SHARD(0, 1, kShardRecv);
  else if (pow2) SSPD_SHARD(0, 0, kShardRecv);
  else if (hist) SSPD_SHARD(1, 1, kShardRecv);
  else SSPD_SHARD(1, 0, kShardRecv);
#undef SSPD_SHARD
  return check_launch();
}
}  // namespace

namespace {
sspd_status shard_relay_locked(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n, const ShardSegs& segs);
}

sspd_status sspd_shard_relay(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n) {
  std::lock_guard<std::mutex> lk(g->mu);
  return shard_relay_locked(g, dev_pairs, n, ShardSegs{});
}

sspd_status sspd_shard_relay_regions(sspd_grid* g, const uint32_t* dev_base, uint64_t region_stride,
                                     const uint64_t* counts, uint32_t n_regions) {
  if (n_regions > 32) return fail(SSPD_INVALID_ARGUMENT, "shard_relay_regions: at most 32 regions");
  ShardSegs segs{};
  segs.stride = region_stride;
  segs.nseg = n_regions;
  segs.start[0] = 0;
  for (uint32_t i = 0; i < n_regions; ++i) {
    if (counts[i] > region_stride) return fail(SSPD_INVALID_ARGUMENT, "shard_relay_regions: count past the region");
    segs.start[i + 1] = segs.start[i] + counts[i];
  }
  for (uint32_t i = n_regions + 1; i < 33; ++i) segs.start[i] = ~0ull;  // the segment search never runs past nseg
  std::lock_guard<std::mutex> lk(g->mu);
  return shard_relay_locked(g, dev_base, segs.start[n_regions], segs);
}

sspd_status sspd_shard_relay_regions_dev(sspd_grid* g, const uint32_t* dev_base, uint64_t region_stride,
                                         const uint64_t* dev_counts, uint64_t count_stride, uint32_t n_regions) {
  if (n_regions == 0 || n_regions > 32 || !dev_counts)
    return fail(SSPD_INVALID_ARGUMENT, "shard_relay_regions: 1..32 regions and device counts");
  std::lock_guard<std::mutex> lk(g->mu);
  if (!g->shard_ovf.p) return fail(SSPD_INVALID_ARGUMENT, "shard_relay: not a relayed sharded grid");
  return shard_relay_locked(g, dev_base, region_stride * n_regions,
                            dev_segs(g, region_stride, dev_counts, count_stride, n_regions, ~0u));
}

namespace {
sspd_status shard_relay_locked(sspd_grid* g, const uint32_t* dev_pairs, uint64_t n, const ShardSegs& segs) {
  if (n == 0) return SSPD_OK;
  DeviceGuard dg(g->device);
  if (!g->shard || !g->relay) return fail(SSPD_INVALID_ARGUMENT, "shard_relay: not a relayed sharded grid");
  sspd_status ps = ensure_pairset_locked(g);  // sizes the relay set too
  if (ps) return ps;
  if (!g->relayset.p) {  // same size as the pair set: the pair owner's share of the routers' union
    if (g->relayset.ensure((g->pairset_mask + 1) * 8) != cudaSuccess)
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (relay set)");
    CU(cudaMemsetAsync(g->relayset.p, 0xff, g->relayset.bytes, g->stream));
  }
  g->pristine = false;
  g->relayset_dirty = true;
  const bool pow2 = (g->eta & (g->eta - 1)) == 0 && g->eta <= (1u << 31);
  const bool hist = g->K && g->hist_valid;
  const unsigned blocks = grid_blocks(g, (n + 3) / 4, 256, SSPD_SCAN_BLOCKS_PER_SM);
  auto* tb = g->relayset.as<unsigned long long>();
  const uint64_t mask = (g->relayset.bytes / 8) - 1;
  Prof p(g, "scan", n);
#define SSPD_RELAY(H1, HI)                                                                                    \
  scan_shard_kernel<H1, HI, kShardOwn><<<blocks, 256, 0, g->stream>>>(dev_pairs, n, g->d_tabs, g->geo, tb, mask, \
                                                                      g->stamps, g->now, g->hist, g->K, g->shard_b, \
                                                                      segs)
  if (pow2 && hist) SSPD_RELAY(0, 1);
  else if (pow2) SSPD_RELAY(0, 0);
  else if (hist) SSPD_RELAY(1, 1);
  else SSPD_RELAY(1, 0);
#undef SSPD_RELAY
  return check_launch();
}
}  // namespace

sspd_status sspd_shard_hot(sspd_grid* g, uint32_t k, uint64_t cutoff, uint32_t** dev_hot_words, uint64_t* n_words) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (!g->shard) return fail(SSPD_INVALID_ARGUMENT, "shard_hot: not a sharded grid");
  sspd_status s = hot_locked(g, k, cutoff, nullptr, nullptr, false);
  if (s) return s;
  CU(cudaStreamSynchronize(g->stream));
  *dev_hot_words = g->hot_words.as<uint32_t>();
  *n_words = (uint64_t)g->r * (((1u << g->q) + 31) / 32);
  return SSPD_OK;
}

sspd_status sspd_shard_select(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap, uint64_t* n_surv,
                              uint32_t** dev_masks, uint64_t* mask_words, uint32_t* ovf_level, uint64_t* ovf_count) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  *n_surv = 0;
  *mask_words = 0;
  *dev_masks = nullptr;
  if (!g->shard) return fail(SSPD_INVALID_ARGUMENT, "shard_select: not a sharded grid");
  if (sspd_status s = no_pending(g, "shard_select")) return s;
  if (g->r > 64) return fail(SSPD_INVALID_ARGUMENT, "reconstruct: r > 64 unsupported");
  for (int attempt = 0;; ++attempt) {
    uint64_t C = 0;
    RecStep step;
    sspd_status s = recon_attempt(g, k, cutoff, cap, true, false, &C, &step, ovf_level, ovf_count);
    if (s) return s;
    if (step == RecStep::kEmptyRow) return SSPD_OK;
    if (step == RecStep::kRetry) {
      if (attempt > 8) return fail(SSPD_CUDA_ERROR, "reconstruct: candidate buffer did not converge");
      continue;
    }
    const uint64_t ns = g->meta_host->surv;
    const uint32_t W = (g->eta + 31) / 32;
    if (g->masks.ensure(std::max<uint64_t>(ns * W, 1) * 4) != cudaSuccess)
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (survivor masks)");
    if (ns) {
      // The joins append survivors in a timing-dependent order, so each
      // router's list is put in one canonical order -- by cip, which fixes
      // the whole tuple (rhfg) -- before the masks are AND-ed index by index.
      uint32_t* s_idx = g->surv.as<uint32_t>();
      std::vector<uint32_t> idx(ns), cip(ns), order(ns);
      CU(cudaMemcpyAsync(idx.data(), s_idx, ns * 4, cudaMemcpyDeviceToHost, g->stream));
      CU(cudaMemcpyAsync(cip.data(), s_idx + C, ns * 4, cudaMemcpyDeviceToHost, g->stream));
      CU(cudaStreamSynchronize(g->stream));
      for (uint64_t i = 0; i < ns; ++i) order[i] = (uint32_t)i;
      std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cip[a] < cip[b]; });
      std::vector<uint32_t> idx2(ns), cip2(ns);
      for (uint64_t i = 0; i < ns; ++i) {
        idx2[i] = idx[order[i]];
        cip2[i] = cip[order[i]];
      }
      CU(cudaMemcpyAsync(s_idx, idx2.data(), ns * 4, cudaMemcpyHostToDevice, g->stream));
      CU(cudaMemcpyAsync(s_idx + C, cip2.data(), ns * 4, cudaMemcpyHostToDevice, g->stream));
      g->d2h_bytes += ns * 8;
      g->h2d_bytes += ns * 8;
      Prof p(g, "finalize", ns * W);
      shard_mask_kernel<<<grid_blocks(g, ns * W, 256, 8), 256, 0, g->stream>>>(
          g->last_tuples->as<uint32_t>(), g->stamps, g->geo, g->now - (k <= 0xFFFFu ? k : 0u), kmode_of(k),
          g->meta.as<ReconMeta>(), g->surv.as<uint32_t>(), g->shard_args.world, g->shard_args.rank,
          g->masks.as<uint32_t>());
      s = check_launch();
      if (s) return s;
    }
    CU(cudaStreamSynchronize(g->stream));
    g->surv_cap = C;
    *n_surv = ns;
    *dev_masks = g->masks.as<uint32_t>();
    *mask_words = ns * W;
    return SSPD_OK;
  }
}

sspd_status sspd_shard_finish(sspd_grid* g, uint64_t cutoff, sspd_detection* out, uint64_t out_cap,
                              uint64_t* n_out) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  *n_out = 0;
  if (!g->shard) return fail(SSPD_INVALID_ARGUMENT, "shard_finish: not a sharded grid");
  const uint64_t ns = g->meta_host->surv;
  if (ns == 0) return SSPD_OK;
  const uint64_t C = g->surv_cap;
  uint32_t* s_idx = g->surv.as<uint32_t>();
  {
    Prof p(g, "finalize", ns);
    shard_popcount_kernel<<<grid_blocks(g, ns * 32, 256, 4), 256, 0, g->stream>>>(
        g->masks.as<uint32_t>(), g->meta.as<ReconMeta>(), (g->eta + 31) / 32, s_idx + 2 * C);
  }
  sspd_status s = check_launch();
  if (s) return s;
  std::vector<uint32_t> cip(ns), rk(ns);
  CU(cudaMemcpyAsync(cip.data(), s_idx + C, ns * 4, cudaMemcpyDeviceToHost, g->stream));
  CU(cudaMemcpyAsync(rk.data(), s_idx + 2 * C, ns * 4, cudaMemcpyDeviceToHost, g->stream));
  CU(cudaStreamSynchronize(g->stream));
  g->d2h_bytes += ns * 8;
  report(g, cip, rk, cutoff, out, out_cap, n_out);
  return SSPD_OK;
}

sspd_status sspd_merge(const sspd_grid* const* grids_c, uint64_t n, int policy, sspd_grid* out) {
  if (n == 0) return fail(SSPD_INVALID_ARGUMENT, "merge_rseas: empty set");
  auto** grids = const_cast<sspd_grid**>(grids_c);
  for (uint64_t i = 0; i < n; ++i)
    if (sspd_status w = wide_only(grids[i], "merge_rseas")) return w;
  if (sspd_status w = wide_only(out, "merge_rseas")) return w;
  for (uint64_t i = 0; i < n; ++i)
    if (sspd_status w = whole_only(grids[i], "merge_rseas")) return w;
  if (sspd_status w = whole_only(out, "merge_rseas")) return w;
  for (uint64_t i = 0; i < n; ++i)
    if (!compatible(grids[i], grids[0]))
      return fail(SSPD_INVALID_ARGUMENT, "merge_rseas: incompatible snapshots (seed/q/r/delta/eta differ)");
  if (!compatible(out, grids[0]))
    return fail(SSPD_INVALID_ARGUMENT, "merge_rseas: incompatible snapshots (seed/q/r/delta/eta differ)");
  // fold pending touches of every input, and quiesce their streams
  uint32_t now_common = 0;
  for (uint64_t i = 0; i < n; ++i) {
    std::lock_guard<std::mutex> lk(grids[i]->mu);
    DeviceGuard dg(grids[i]->device);
    sspd_status s = commit_locked(grids[i]);
    if (s) return s;
    CU(cudaStreamSynchronize(grids[i]->stream));
    now_common = std::max(now_common, grids[i]->now);
  }
  bool out_is_input = false;
  for (uint64_t i = 0; i < n; ++i) out_is_input |= grids[i] == out;
  std::unique_lock<std::mutex> lk(out->mu, std::defer_lock);
  if (!out_is_input) lk.lock();
  DeviceGuard dg(out->device);
  if (!out_is_input) {
    sspd_status s = commit_locked(out);
    if (s) return s;
  }
  {
    sspd_status s = pairset_reset_locked(out);
    if (s) return s;
  }
  // Peer access for inputs on other devices (NVLink loads in merge_kernel).
  std::vector<MergeSrc> srcs(n);
  for (uint64_t i = 0; i < n; ++i) {
    if (grids[i]->device != out->device) {
      cudaError_t e = cudaDeviceEnablePeerAccess(grids[i]->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(SSPD_CUDA_ERROR, std::string("CUDA error: peer access: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
    srcs[i] = MergeSrc{grids[i]->stamps, now_common - grids[i]->now};
  }
  const size_t sbytes = n * sizeof(MergeSrc);
  ScopedBuf tmp;
  if (tmp.ensure(sbytes) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (merge)");
  CU(cudaMemcpyAsync(tmp.p, srcs.data(), sbytes, cudaMemcpyHostToDevice, out->stream));
  out->h2d_bytes += (sbytes);
  {
    Prof p(out, "merge", out->geo.n_rec * n);
    merge_kernel<<<grid_blocks(out, out->geo.n_rec / 4 + 1, 256, 8), 256, 0, out->stream>>>(
        tmp.as<MergeSrc>(), (uint32_t)n, out->geo.n_rec, now_common, policy == SSPD_UNION_MIN ? 1 : 0,
        out->stamps);
  }
  sspd_status s = check_launch();
  CU(cudaStreamSynchronize(out->stream));
  if (s) return s;
  out->now = now_common;
  out->hist_valid = false;
  out->pristine = false;
  return SSPD_OK;
}

sspd_status sspd_equal(sspd_grid* a, sspd_grid* b, int* equal) {
  if (sspd_status w = whole_only(a, "==")) return w;
  if (sspd_status w = whole_only(b, "==")) return w;
  *equal = 0;
  if (sspd_status w = wide_only(a, "operator==")) return w;
  if (sspd_status w = wide_only(b, "operator==")) return w;
  if (a->geo.n_rec != b->geo.n_rec) return SSPD_OK;
  for (sspd_grid* g : {a, b}) {
    std::lock_guard<std::mutex> lk(g->mu);
    DeviceGuard dg(g->device);
    sspd_status s = commit_locked(g);
    if (s) return s;
    CU(cudaStreamSynchronize(g->stream));
  }
  std::lock_guard<std::mutex> lk(a->mu);
  DeviceGuard dg(a->device);
  if (b->device != a->device) {
    cudaError_t e = cudaDeviceEnablePeerAccess(b->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return fail(SSPD_CUDA_ERROR, std::string("CUDA error: peer access: ") + cudaGetErrorString(e));
    cudaGetLastError();
  }
  int* flag = static_cast<int*>(pinned_scratch(a));
  if (a->misc.ensure(64) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
  CU(cudaMemsetAsync(a->misc.p, 0, 4, a->stream));
  {
    Prof p(a, "equal", a->geo.n_rec);
    equal_kernel<<<grid_blocks(a, a->geo.n_rec, 256, 8), 256, 0, a->stream>>>(
        a->stamps, a->now, b->stamps, b->now, a->geo.n_rec, a->misc.as<int>());
  }
  CU(cudaMemcpyAsync(flag, a->misc.p, 4, cudaMemcpyDeviceToHost, a->stream));
  a->d2h_bytes += (4);
  CU(cudaStreamSynchronize(a->stream));
  *equal = *flag ? 0 : 1;
  return check_launch();
}

sspd_status sspd_track_window(sspd_grid* g, uint32_t k_max) {
  if (k_max > 65534) return fail(SSPD_OUT_OF_RANGE, "track_window: k must be in [0, 65534]");
  if (g->width != 32 && k_max == g->K) return SSPD_OK;  // fixed at creation
  if (sspd_status w = wide_only(g, "track_window")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (g->hist) {
    cache_free(g->hist);
    g->hist = nullptr;
  }
  g->K = k_max;
  g->hist_valid = false;
  if (k_max) {
    if (cache_alloc((void**)&g->hist, (size_t)k_max * g->geo.ncells * 4) != cudaSuccess) {
      cudaGetLastError();
      g->K = 0;
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (window ring)");
    }
    if (g->pristine) {  // nothing seen yet: the ring is all zero, no pass over the stamps
      CU(cudaMemsetAsync(g->hist, 0, (size_t)k_max * g->geo.ncells * 4, g->stream));
      g->hist_valid = true;
      return SSPD_OK;
    }
    return hist_rebuild_locked(g);
  }
  return SSPD_OK;
}

sspd_status sspd_grid_stamps(sspd_grid* g, uint32_t** dev_stamps, uint64_t* words) {
  if (sspd_status w = whole_only(g, "grid_stamps")) return w;
  if (sspd_status w = wide_only(g, "grid_stamps")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  s = pairset_reset_locked(g);
  if (s) return s;
  CU(cudaStreamSynchronize(g->stream));
  *dev_stamps = g->stamps;
  *words = g->geo.n_rec;
  // the caller may rewrite stamps (e.g. an in-place NCCL max); the ring is
  // rebuilt from them on next use
  g->hist_valid = false;
  g->pristine = false;
  return SSPD_OK;
}

sspd_status sspd_set_exchange(sspd_grid* g, int mode) {
  if (mode != 0) {
    if (sspd_status w = wide_only(g, "set_exchange")) return w;
    if (sspd_status w = whole_only(g, "set_exchange")) return w;
  }
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (mode == 1)
    if (sspd_status ts = ensure_touched_locked(g)) return ts;
  g->record_touched = mode == 1;
  g->export_pairs = mode == 2;
  return SSPD_OK;
}

sspd_status sspd_set_push(sspd_grid* g, void* dev_peer_ptrs, uint32_t world, uint32_t rank, uint64_t region_cap) {
  if (sspd_status w = whole_only(g, "set_push")) return w;
  if (world > 1)
    if (sspd_status w = wide_only(g, "set_push")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  if (world > 1 && (!dev_peer_ptrs || rank >= world || region_cap == 0))
    return fail(SSPD_INVALID_ARGUMENT, "set_push: bad peer table");
  g->push = PushArgs{static_cast<uint2* const*>(dev_peer_ptrs), world, rank, region_cap};
  return SSPD_OK;
}

sspd_status sspd_grid_new_pairs(sspd_grid* g, uint32_t** dev_pairs, uint64_t* count) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  uint64_t c = 0;
  if (g->newpairs_count.p) {
    CU(cudaMemcpyAsync(pinned_scratch(g), g->newpairs_count.p, 8, cudaMemcpyDeviceToHost, g->stream));
    CU(cudaStreamSynchronize(g->stream));
    c = *static_cast<uint64_t*>(pinned_scratch(g));
  }
  *dev_pairs = g->newpairs.as<uint32_t>();
  *count = c;
  return SSPD_OK;
}

sspd_status sspd_checked_status(int device, uint32_t* first_line, uint64_t* failures, int reset) {
  *first_line = 0;
  *failures = 0;
#ifdef SSPD_CHECKED
  DeviceGuard dg(device);
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpyFromSymbol(first_line, g_chk_line, sizeof(uint32_t)));
  unsigned long long n = 0;
  CU(cudaMemcpyFromSymbol(&n, g_chk_count, sizeof n));
  *failures = n;
  if (reset) {
    const uint32_t z = 0;
    const unsigned long long z8 = 0;
    CU(cudaMemcpyToSymbol(g_chk_line, &z, sizeof z));
    CU(cudaMemcpyToSymbol(g_chk_count, &z8, sizeof z8));
  }
  return SSPD_OK;
#else
  (void)device;
  (void)reset;
  return fail(SSPD_INVALID_ARGUMENT, "checked_status: not a checked build (lib/libsspd_cuda_checked.so)");
#endif
}

sspd_status sspd_grid_fresh_pairs(sspd_grid* g, uint64_t* count) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  uint64_t c = 0;
  if (g->fresh_count.p) {
    CU(cudaMemcpyAsync(pinned_scratch(g), g->fresh_count.p, 8, cudaMemcpyDeviceToHost, g->stream));
    CU(cudaStreamSynchronize(g->stream));
    c = *static_cast<uint64_t*>(pinned_scratch(g));
  }
  *count = c;
  return SSPD_OK;
}

sspd_status sspd_grid_keyset(sspd_grid* g, uint32_t** dev_entries, uint32_t* log2_entries) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  CU(cudaStreamSynchronize(g->stream));
  if (dev_entries) *dev_entries = g->cset.as<uint32_t>();
  if (log2_entries) *log2_entries = g->cset.p ? g->cset_lg : 0;
  return SSPD_OK;
}

sspd_status sspd_scan_mode(sspd_grid* g, int mode, int filter) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (mode >= -1 && mode <= 3) g->scan_mode = mode;
  if (filter >= 0) g->scan_filter = filter != 0;
  return SSPD_OK;
}

sspd_status sspd_grid_touched(sspd_grid* g, uint32_t** dev_bits, uint64_t* words) {
  if (sspd_status w = wide_only(g, "grid_touched")) return w;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  if (sspd_status ts = ensure_touched_locked(g)) return ts;
  CU(cudaStreamSynchronize(g->stream));
  *dev_bits = g->touched;
  *words = g->n_words;
  return SSPD_OK;
}

sspd_status sspd_grid_io_bytes(sspd_grid* g, uint64_t* h2d, uint64_t* d2h, int reset) {
  std::lock_guard<std::mutex> lk(g->mu);
  if (h2d) *h2d = g->h2d_bytes;
  if (d2h) *d2h = g->d2h_bytes;
  if (reset) g->h2d_bytes = g->d2h_bytes = 0;
  return SSPD_OK;
}

sspd_status sspd_profile_enable(sspd_grid* g, int on) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  g->profiling = on != 0;
  // events for a few hundred launches up front, so profiling adds only
  // cudaEventRecord calls to the timed work
  while (g->profiling && g->event_pool.size() < 512) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    g->event_pool.push_back(e);
  }
  return SSPD_OK;
}

sspd_status sspd_profile_reset(sspd_grid* g) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  cudaStreamSynchronize(g->stream);
  for (auto& r : g->prof) {
    g->event_pool.push_back(r.a);
    g->event_pool.push_back(r.b);
  }
  g->prof.clear();
  return SSPD_OK;
}

sspd_status sspd_profile_read(sspd_grid* g, const char* kernel, double* total_ms, uint64_t* launches,
                              uint64_t* units) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  CU(cudaStreamSynchronize(g->stream));
  double ms = 0;
  uint64_t cnt = 0, u = 0;
  for (auto& r : g->prof) {
    if (kernel && std::strcmp(kernel, r.name) != 0) continue;
    float t = 0;
    CU(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    ++cnt;
    u += r.units;
  }
  if (total_ms) *total_ms = ms;
  if (launches) *launches = cnt;
  if (units) *units = u;
  return SSPD_OK;
}

sspd_status sspd_exact_counts(int device, const uint32_t* const* dev_segments, const uint64_t* seg_pairs,
                              uint32_t n_segments, uint64_t distinct_hint, uint32_t min_count, uint32_t* cips,
                              uint32_t* counts, uint64_t out_cap, uint64_t* n_out, void* cuda_stream) {
  *n_out = 0;
  uint64_t total = 0;
  for (uint32_t i = 0; i < n_segments; ++i) total += seg_pairs[i];
  const uint64_t want = std::max<uint64_t>(distinct_hint ? distinct_hint : total, 1024);
  uint64_t pe = 1;
  while (pe < 2 * want) pe <<= 1;
  uint64_t ce = 1;
  while (ce < 2 * std::min<uint64_t>(want, 1ull << 32)) ce <<= 1;
  DeviceGuard dg(device);
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  ScopedBuf pset, ckeys, ccounts, flags, out;
  if (pset.ensure(pe * 8) != cudaSuccess || ckeys.ensure(ce * 8) != cudaSuccess ||
      ccounts.ensure(ce * 4) != cudaSuccess || flags.ensure(64) != cudaSuccess ||
      out.ensure(std::max<uint64_t>(out_cap, 1) * 8 + 64) != cudaSuccess) {
    cudaGetLastError();
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (exact counts)");
  }
  CU(cudaMemsetAsync(pset.p, 0xff, pe * 8, st));
  CU(cudaMemsetAsync(ckeys.p, 0, ce * 8, st));
  CU(cudaMemsetAsync(ccounts.p, 0, ce * 4, st));
  CU(cudaMemsetAsync(flags.p, 0, 64, st));
  const unsigned blocks = (unsigned)sm_count(device) * 8;
  for (uint32_t i = 0; i < n_segments; ++i) {
    if (!seg_pairs[i]) continue;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    exact_insert_kernel<<<blocks, 256, 0, st>>>(dev_segments[i], seg_pairs[i], pset.as<unsigned long long>(),
                                                pe - 1, ckeys.as<unsigned long long>(), ccounts.as<uint32_t>(),
                                                ce - 1, flags.as<unsigned int>());
  }
  auto* counter = reinterpret_cast<unsigned long long*>(static_cast<char*>(flags.p) + 32);
  uint32_t* o_cip = out.as<uint32_t>();
  uint32_t* o_cnt = o_cip + std::max<uint64_t>(out_cap, 1);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  exact_emit_kernel<<<blocks, 256, 0, st>>>(ckeys.as<unsigned long long>(), ccounts.as<uint32_t>(), ce, min_count,
                                            o_cip, o_cnt, out_cap, counter);
  sspd_status s = check_launch();
  if (s) return s;
  uint32_t host_flags[16] = {0};
  CU(cudaMemcpyAsync(host_flags, flags.p, 64, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (host_flags[0]) return fail(SSPD_OUT_OF_RANGE, "exact_counts: table full (raise distinct_hint)");
  uint64_t cnt = 0;
  std::memcpy(&cnt, reinterpret_cast<char*>(host_flags) + 32, 8);
  *n_out = cnt;
  const uint64_t m = std::min(cnt, out_cap);
  if (m) {
    std::vector<uint32_t> a(m), b(m);
    CU(cudaMemcpyAsync(a.data(), o_cip, m * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(b.data(), o_cnt, m * 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    std::vector<uint64_t> order(m);
    for (uint64_t i = 0; i < m; ++i) order[i] = (uint64_t)a[i] << 32 | b[i];
    std::sort(order.begin(), order.end());  // ascending cip, like the reference's sorted tables
    for (uint64_t i = 0; i < m; ++i) {
      cips[i] = (uint32_t)(order[i] >> 32);
      counts[i] = (uint32_t)order[i];
    }
  }
  return SSPD_OK;
}

static_assert(sizeof(sspd_synth_params_t) == sizeof(sspd_synth_params), "synth params layout");

__global__ void synth_kernel(sspd_synth_params p, const uint64_t* __restrict__ cdf, uint64_t slot,
                             uint64_t j0, uint64_t n, uint2* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c, o;
    sspd_synth_pair(&p, cdf, slot, j0 + i, &c, &o);
    out[i] = make_uint2(c, o);
  }
}

sspd_status sspd_synth_zipf_cdf(uint32_t hosts, double exponent, uint64_t* cdf_out) {
  if (hosts == 0) return fail(SSPD_INVALID_ARGUMENT, "synth: hosts == 0");
  std::vector<double> acc(hosts);
  double s = 0;
  for (uint32_t i = 0; i < hosts; ++i) {
    s += std::pow(static_cast<double>(i + 1), -exponent);
    acc[i] = s;
  }
  const double scale = 9223372036854775808.0;  // 2^63
  for (uint32_t i = 0; i < hosts; ++i) {
    const double v = acc[i] / s * scale;
    cdf_out[i] = v >= scale ? (1ull << 63) : static_cast<uint64_t>(v);
  }
  cdf_out[hosts - 1] = 1ull << 63;
  return SSPD_OK;
}

static bool synth_ok(const sspd_synth_params_t* p) {
  return p && p->hosts && p->n_shards && p->shard < p->n_shards &&
         (p->n_super == 0 || p->super_fanout);
}

sspd_status sspd_synth_host(const sspd_synth_params_t* p, const uint64_t* cdf, uint64_t slot, uint64_t j0,
                            uint64_t n, uint32_t* pairs_out) {
  if (!synth_ok(p)) return fail(SSPD_INVALID_ARGUMENT, "synth: bad parameters");
  const auto* q = reinterpret_cast<const sspd_synth_params*>(p);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)n; ++i)
    sspd_synth_pair(q, cdf, slot, j0 + (uint64_t)i, &pairs_out[2 * i], &pairs_out[2 * i + 1]);
  return SSPD_OK;
}

sspd_status sspd_synth_device(int device, const sspd_synth_params_t* p, const uint64_t* dev_cdf, uint64_t slot,
                              uint64_t j0, uint64_t n, uint32_t* dev_pairs_out, void* cuda_stream) {
  if (!synth_ok(p)) return fail(SSPD_INVALID_ARGUMENT, "synth: bad parameters");
  DeviceGuard dg(device);
  const auto q = *reinterpret_cast<const sspd_synth_params*>(p);
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148ull * 16));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  synth_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(cuda_stream)>>>(q, dev_cdf, slot, j0, n,
                                                                           reinterpret_cast<uint2*>(dev_pairs_out));
  return check_launch();
}

uint32_t sspd_synth_super_cip(const sspd_synth_params_t* p, uint32_t i) {
  return sspd_super_cip(reinterpret_cast<const sspd_synth_params*>(p), i);
}

}  // extern "C"
