// sspd_cuda.cu -- C ABI (include/sspd_cuda.h) over the sm_100a kernels in
// kernels.cuh.  Host orchestration only: argument checks with the
// reference's error texts, per-grid streams and scratch, chunked host->device
// copies, and the bits of reconstruction that are inherently host-side
// (dedup + sort of the reported hosts, estimate_cardinality in double).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sspd_cuda.h"
#include "kernels.cuh"
#include "synth.h"

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

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
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
  HashTabs* d_tabs = nullptr;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};
  DevBuf stage[2];       // host pair staging
  DevBuf counts, hot_cols, hot_rowcnt, hotT, tupA, tupB, fin, misc;
  void* pinned_small = nullptr;  // 4 KB pinned scratch for counters
  bool profiling = false;
  std::vector<ProfRec> prof;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic, for e2e accounting
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
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// Persistent-style grid size: a multiple of the SM count.
unsigned grid_blocks(const sspd_grid* g, uint64_t work_items, unsigned threads, unsigned per_sm) {
  const uint64_t need = (work_items + threads - 1) / threads;
  const uint64_t cap = (uint64_t)sm_count(g->device) * per_sm;
  return (unsigned)std::max<uint64_t>(1, std::min(need, cap));
}

struct Prof {
  sspd_grid* g;
  ProfRec rec{};
  Prof(sspd_grid* g_, const char* name, uint64_t units) : g(g_) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g->profiling) return;
    rec.name = name;
    rec.units = units;
    cudaEventCreate(&rec.a);
    cudaEventCreate(&rec.b);
    cudaEventRecord(rec.a, g->stream);
  }
  ~Prof() {
    if (!g->profiling) return;
    cudaEventRecord(rec.b, g->stream);
    g->prof.push_back(rec);
  }
};

sspd_status check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SSPD_CUDA_ERROR, std::string("CUDA launch: ") + cudaGetErrorString(e));
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
  if (g->K && k <= g->K) {
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
sspd_status hot_locked(sspd_grid* g, uint32_t k, uint64_t cutoff, std::vector<uint32_t>& host_rowcnt) {
  sspd_status s = counts_locked(g, k);
  if (s) return s;
  const uint32_t ncol = 1u << g->q;
  const uint32_t wpk = words_per_key(g);
  const size_t t_words = (size_t)g->r * ((size_t)wpk << (g->q - g->delta));
  if (g->hot_cols.ensure((size_t)g->r * ncol * 4) != cudaSuccess ||
      g->hot_rowcnt.ensure((size_t)g->r * 4) != cudaSuccess || g->hotT.ensure(t_words * 4) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (hot sets)");
  CU(cudaMemsetAsync(g->hotT.p, 0, t_words * 4, g->stream));
  {
    Prof p(g, "hot_compact", g->geo.ncells);
    hot_compact_kernel<<<g->r, 1024, 0, g->stream>>>(g->counts.as<uint32_t>(), g->geo, cutoff,
                                                     g->hot_cols.as<uint32_t>(),
                                                     g->hot_rowcnt.as<uint32_t>(), g->hotT.as<uint32_t>(),
                                                     wpk);
  }
  s = check_launch();
  if (s) return s;
  host_rowcnt.resize(g->r);
  CU(cudaMemcpyAsync(host_rowcnt.data(), g->hot_rowcnt.p, g->r * 4, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (g->r * 4);
  CU(cudaStreamSynchronize(g->stream));
  return SSPD_OK;
}

// estimate_cardinality (estimator.cpp:25-30), host double arithmetic.
double estimate(uint64_t eta, uint64_t r_k) {
  const uint64_t z0 = eta - r_k;
  const double deta = static_cast<double>(eta);
  if (z0 == 0) return deta * std::log(deta);
  return -deta * std::log(static_cast<double>(z0) / deta);
}

sspd_status finalize_dev(sspd_grid* g, const uint32_t* d_tuples, uint64_t n, uint32_t k, uint64_t cutoff,
                         uint8_t* d_accepted, std::vector<uint32_t>* idx, std::vector<uint32_t>* cips,
                         std::vector<uint32_t>* rks) {
  // fin buffer: counter (8B) + 3 arrays of n u32
  const size_t bytes = 256 + (size_t)std::max<uint64_t>(n, 1) * 12;
  if (g->fin.ensure(bytes) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (finalize)");
  auto* counter = reinterpret_cast<unsigned long long*>(g->fin.p);
  uint32_t* o_idx = reinterpret_cast<uint32_t*>(static_cast<char*>(g->fin.p) + 256);
  uint32_t* o_cip = o_idx + n;
  uint32_t* o_rk = o_cip + n;
  CU(cudaMemsetAsync(counter, 0, 8, g->stream));
  if (n) {
    const unsigned blocks = grid_blocks(g, n * 32, 256, 8);
    Prof p(g, "finalize", n);
    finalize_kernel<<<blocks, 256, 0, g->stream>>>(d_tuples, n, g->stamps, g->d_tabs, g->geo, g->now - k,
                                                   cutoff, o_idx, o_cip, o_rk, counter, d_accepted);
    sspd_status s = check_launch();
    if (s) return s;
  }
  unsigned long long cnt = 0;
  CU(cudaMemcpyAsync(&cnt, counter, 8, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (8);
  CU(cudaStreamSynchronize(g->stream));
  if (idx) {
    idx->resize(cnt);
    cips->resize(cnt);
    rks->resize(cnt);
    if (cnt) {
      CU(cudaMemcpyAsync(idx->data(), o_idx, cnt * 4, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (cnt * 4);
      CU(cudaMemcpyAsync(cips->data(), o_cip, cnt * 4, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (cnt * 4);
      CU(cudaMemcpyAsync(rks->data(), o_rk, cnt * 4, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (cnt * 4);
      CU(cudaStreamSynchronize(g->stream));
    }
  }
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

sspd_status sspd_grid_create(int device, uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta,
                             sspd_grid** out) {
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
  g->geo.eta_shift = (eta & (eta - 1)) == 0 ? (uint32_t)__builtin_ctz(eta) : 0xFFu;
  g->geo.ncells = r << q;
  g->geo.n_rec = (uint64_t)g->geo.ncells * eta;
  g->by_eta = Div40::make(eta);
  g->n_words = (g->geo.n_rec + 31) / 32;
  auto cleanup = [&](const std::string& why) {
    sspd_grid_destroy(g);
    return fail(SSPD_CUDA_ERROR, why);
  };
  if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup("CUDA error: stream creation failed");
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&g->ev_copy[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_used[i], cudaEventDisableTiming);
  }
  if (cudaMalloc(&g->stamps, g->geo.n_rec * 4) != cudaSuccess) {
    cudaGetLastError();
    return cleanup("CUDA error: out of memory allocating " + std::to_string(g->geo.n_rec * 4) +
                   " bytes of stamps");
  }
  if (cudaMalloc(&g->touched, g->n_words * 4) != cudaSuccess) {
    cudaGetLastError();
    return cleanup("CUDA error: out of memory allocating the touched bitmap");
  }
  if (cudaMalloc(&g->d_tabs, sizeof(HashTabs)) != cudaSuccess) return cleanup("CUDA error: tables");
  if (cudaMallocHost(&g->pinned_small, 4096) != cudaSuccess) return cleanup("CUDA error: pinned scratch");
  HashTabs h = make_tabs(seed);
  if (cudaMemcpyAsync(g->d_tabs, &h, sizeof h, cudaMemcpyHostToDevice, g->stream) != cudaSuccess)
    return cleanup("CUDA error: table upload");
  // All recorders never seen: stamp 0.
  if (cudaMemsetAsync(g->stamps, 0, g->geo.n_rec * 4, g->stream) != cudaSuccess ||
      cudaMemsetAsync(g->touched, 0, g->n_words * 4, g->stream) != cudaSuccess)
    return cleanup("CUDA error: grid init");
  if (cudaStreamSynchronize(g->stream) != cudaSuccess) return cleanup("CUDA error: grid init sync");
  *out = g;
  return SSPD_OK;
}

sspd_status sspd_grid_destroy(sspd_grid* g) {
  if (!g) return SSPD_OK;
  {
    DeviceGuard dg(g->device);
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->copy_stream) cudaStreamSynchronize(g->copy_stream);
    cudaFree(g->stamps);
    cudaFree(g->touched);
    cudaFree(g->hist);
    cudaFree(g->d_tabs);
    if (g->pinned_small) cudaFreeHost(g->pinned_small);
    for (DevBuf* b : {&g->stage[0], &g->stage[1], &g->counts, &g->hot_cols, &g->hot_rowcnt, &g->hotT,
                      &g->tupA, &g->tupB, &g->fin, &g->misc})
      b->release();
    for (auto& r : g->prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
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
  auto* src = const_cast<sspd_grid*>(src_c);
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
    if (src->K) {
      g->K = src->K;
      CU(cudaMalloc(&g->hist, (size_t)g->K * g->geo.ncells * 4));
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

sspd_status sspd_grid_synchronize(sspd_grid* g) {
  DeviceGuard dg(g->device);
  CU(cudaStreamSynchronize(g->stream));
  return SSPD_OK;
}

sspd_status sspd_scan(sspd_grid* g, const uint32_t* pairs, uint64_t n, int pairs_on_device) {
  if (n == 0) return SSPD_OK;
  if (!pairs) return fail(SSPD_INVALID_ARGUMENT, "scan_batch: null pairs");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  const bool pow2 = (g->eta & (g->eta - 1)) == 0;
  auto launch = [&](const uint32_t* dp, uint64_t cnt) {
    const unsigned blocks = grid_blocks(g, (cnt + 3) / 4, 256, 8);
    Prof p(g, "scan", cnt);
    if (pow2)
      scan_bitmap_kernel<0><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, g->touched);
    else
      scan_bitmap_kernel<1><<<blocks, 256, 0, g->stream>>>(dp, cnt, g->d_tabs, g->geo, g->touched);
  };
  g->pending = true;
  if (pairs_on_device) {
    launch(pairs, n);
    return check_launch();
  }
  // Host pairs: double-buffered chunks; the copy stream fills one staging
  // buffer while the scan consumes the other.
  const uint64_t chunk = 8ull << 20;  // pairs per chunk (64 MiB)
  const uint64_t chunk_pairs = std::min<uint64_t>(chunk, n);
  for (int i = 0; i < 2; ++i)
    if (g->stage[i].ensure(chunk_pairs * 8) != cudaSuccess)
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (scan staging)");
  uint64_t done = 0;
  int buf = 0;
  // the copy stream must not overwrite staging still read by earlier scans
  CU(cudaEventRecord(g->ev_used[0], g->stream));
  CU(cudaEventRecord(g->ev_used[1], g->stream));
  while (done < n) {
    const uint64_t cnt = std::min(chunk_pairs, n - done);
    CU(cudaStreamWaitEvent(g->copy_stream, g->ev_used[buf], 0));
    CU(cudaMemcpyAsync(g->stage[buf].p, pairs + 2 * done, cnt * 8, cudaMemcpyHostToDevice, g->copy_stream));
  g->h2d_bytes += (cnt * 8);
    CU(cudaEventRecord(g->ev_copy[buf], g->copy_stream));
    CU(cudaStreamWaitEvent(g->stream, g->ev_copy[buf], 0));
    launch(g->stage[buf].as<uint32_t>(), cnt);
    CU(cudaEventRecord(g->ev_used[buf], g->stream));
    done += cnt;
    buf ^= 1;
  }
  // Pageable sources are consumed by the time cudaMemcpyAsync returns; for
  // pinned ones the caller may reuse its buffer only after the copies land.
  CU(cudaStreamSynchronize(g->copy_stream));
  return check_launch();
}

sspd_status sspd_commit(sspd_grid* g) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  g->pending = true;  // the caller may have OR-merged remote touches in
  return commit_locked(g);
}

sspd_status sspd_advance(sspd_grid* g, uint32_t slots) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  for (uint32_t i = 0; i < slots; ++i) {
    if (g->now >= 0x7fffffffu) return fail(SSPD_OUT_OF_RANGE, "advance_slot: slice counter exhausted");
    ++g->now;
    if (g->K && g->hist_valid) {
      // the ring entry of the slot leaving the window becomes `now`'s
      CU(cudaMemsetAsync(g->hist + (uint64_t)(g->now % g->K) * g->geo.ncells, 0, (size_t)g->geo.ncells * 4,
                         g->stream));
    }
  }
  return SSPD_OK;
}

sspd_status sspd_get_distances(sspd_grid* g, uint16_t* host_out, uint64_t offset, uint64_t count) {
  if (offset > g->geo.n_rec || count > g->geo.n_rec - offset)
    return fail(SSPD_OUT_OF_RANGE, "cells: range out of bounds");
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
  if (offset > g->geo.n_rec || count > g->geo.n_rec - offset)
    return fail(SSPD_OUT_OF_RANGE, "cells: range out of bounds");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
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
  return check_launch();
}

sspd_status sspd_active_counts(sspd_grid* g, uint32_t k, uint32_t* host_out) {
  if (k < 1 || k > 65534) return fail(SSPD_OUT_OF_RANGE, "active_count: k must be in [1, 65534]");
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
  if (k < 1 || k > 65534) return fail(SSPD_OUT_OF_RANGE, "active_count: k must be in [1, 65534]");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  std::vector<uint32_t> rc;
  sspd_status s = hot_locked(g, k, cutoff, rc);
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
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (n == 0) return SSPD_OK;
  if (g->tupA.ensure(n * g->r * 4) != cudaSuccess || g->misc.ensure(n) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (finalize)");
  CU(cudaMemcpyAsync(g->tupA.p, tuples, n * g->r * 4, cudaMemcpyHostToDevice, g->stream));
  g->h2d_bytes += (n * g->r * 4);
  std::vector<uint32_t> idx, c, rk;
  s = finalize_dev(g, g->tupA.as<uint32_t>(), n, k, cutoff, g->misc.as<uint8_t>(), &idx, &c, &rk);
  if (s) return s;
  CU(cudaMemcpyAsync(accepted, g->misc.p, n, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (n);
  CU(cudaStreamSynchronize(g->stream));
  for (size_t i = 0; i < idx.size(); ++i) {
    cips[idx[i]] = c[i];
    r_ks[idx[i]] = rk[i];
  }
  return SSPD_OK;
}

sspd_status sspd_reconstruct(sspd_grid* g, uint32_t k, uint64_t cutoff, uint64_t cap, sspd_detection* out,
                             uint64_t out_cap, uint64_t* n_out, uint32_t* ovf_level, uint64_t* ovf_count) {
  if (k < 1 || k > 65534) return fail(SSPD_OUT_OF_RANGE, "active_count: k must be in [1, 65534]");
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  *n_out = 0;
  std::vector<uint32_t> rc;
  sspd_status s = hot_locked(g, k, cutoff, rc);
  if (s) return s;
  for (uint32_t row = 0; row < g->r; ++row)
    if (rc[row] == 0) return SSPD_OK;  // rsea.cpp:173-174
  const uint32_t ncol = 1u << g->q;
  const uint32_t wpk = words_per_key(g);
  const uint64_t t_stride = (uint64_t)wpk << (g->q - g->delta);
  const uint32_t* cols = g->hot_cols.as<uint32_t>();
  const uint32_t* T = g->hotT.as<uint32_t>();
  auto* counter = static_cast<unsigned long long*>(g->pinned_small);  // host copy target
  unsigned long long* d_counter = nullptr;
  if (g->fin.ensure(256) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
  // a dedicated 8-byte device counter lives at the end of the misc buffer
  if (g->misc.ensure(std::max<size_t>(g->misc.bytes, 64)) != cudaSuccess)
    return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory");
  d_counter = reinterpret_cast<unsigned long long*>(g->misc.p);

  // Run one level with growing output capacity; returns survivor count.
  auto run_level = [&](uint32_t m_out, auto&& launch, DevBuf& dst, uint64_t& count) -> sspd_status {
    uint64_t cap_tuples = std::min<uint64_t>(std::max<uint64_t>(dst.bytes / (m_out * 4), 1u << 16), cap);
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (dst.ensure(std::max<uint64_t>(cap_tuples, 1) * m_out * 4) != cudaSuccess)
        return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (candidate buffer)");
      CU(cudaMemsetAsync(d_counter, 0, 8, g->stream));
      launch(dst.as<uint32_t>(), cap_tuples);
      sspd_status e = check_launch();
      if (e) return e;
      CU(cudaMemcpyAsync(counter, d_counter, 8, cudaMemcpyDeviceToHost, g->stream));
  g->d2h_bytes += (8);
      CU(cudaStreamSynchronize(g->stream));
      count = *counter;
      if (count <= cap_tuples || count > cap) return SSPD_OK;
      cap_tuples = count;  // grow and recompute (count <= cap here)
    }
    return SSPD_OK;
  };

  // Level 2 (rsea.cpp:179-201).
  uint64_t n_t = 0;
  {
    const uint64_t pairs = (uint64_t)rc[0] * rc[1];
    s = run_level(
        3,
        [&](uint32_t* dst, uint64_t dcap) {
          const unsigned blocks = grid_blocks(g, pairs, 256, 8);
          Prof p(g, "level2", pairs);
          level2_kernel<<<blocks, 256, 0, g->stream>>>(cols, rc[0], cols + ncol, rc[1], T + 2 * t_stride, wpk,
                                                       g->geo, dst, dcap, d_counter);
        },
        g->tupA, n_t);
    if (s) return s;
    if (n_t > cap) {
      *ovf_level = 2;
      *ovf_count = n_t;
      return fail(SSPD_CANDIDATE_OVERFLOW, "candidate buffer cap exceeded at level 2: " + std::to_string(n_t) +
                                               " tuples, cap " + std::to_string(cap));
    }
  }
  DevBuf* rd = &g->tupA;
  DevBuf* wr = &g->tupB;
  for (uint32_t row = 3; row < g->r; ++row) {
    const uint32_t m = row;  // tuple length before extension
    uint64_t n_next = 0;
    const uint32_t* in = rd->as<uint32_t>();
    const uint64_t n_in = n_t;
    s = run_level(
        m + 1,
        [&](uint32_t* dst, uint64_t dcap) {
          if (!n_in) return;
          const unsigned blocks = grid_blocks(g, n_in, 256, 8);
          Prof p(g, "level_ext", n_in);
          level_ext_kernel<<<blocks, 256, 0, g->stream>>>(in, n_in, m, T + (uint64_t)row * t_stride, wpk, g->geo,
                                                          dst, dcap, d_counter);
        },
        *wr, n_next);
    if (s) return s;
    if (n_next > cap) {
      *ovf_level = row;
      *ovf_count = n_next;
      return fail(SSPD_CANDIDATE_OVERFLOW, "candidate buffer cap exceeded at level " + std::to_string(row) + ": " +
                                               std::to_string(n_next) + " tuples, cap " + std::to_string(cap));
    }
    n_t = n_next;
    std::swap(rd, wr);
  }
  // Finalization + dedup (rsea.cpp:239-254, 112-122).
  std::vector<uint32_t> idx, cip, rk;
  s = finalize_dev(g, rd->as<uint32_t>(), n_t, k, cutoff, nullptr, &idx, &cip, &rk);
  if (s) return s;
  std::map<uint32_t, uint32_t> best;  // cip -> max r_k (estimate is monotone in r_k)
  for (size_t i = 0; i < cip.size(); ++i) {
    auto it = best.emplace(cip[i], rk[i]);
    if (!it.second && rk[i] > it.first->second) it.first->second = rk[i];
  }
  *n_out = best.size();
  uint64_t w = 0;
  for (const auto& [c, r_k] : best) {
    if (w < out_cap) out[w] = sspd_detection{c, r_k, estimate(g->eta, r_k)};
    ++w;
  }
  return SSPD_OK;
}

sspd_status sspd_merge(const sspd_grid* const* grids_c, uint64_t n, int policy, sspd_grid* out) {
  if (n == 0) return fail(SSPD_INVALID_ARGUMENT, "merge_rseas: empty set");
  auto** grids = const_cast<sspd_grid**>(grids_c);
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
  DevBuf tmp;
  if (tmp.ensure(sbytes) != cudaSuccess) return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (merge)");
  CU(cudaMemcpyAsync(tmp.p, srcs.data(), sbytes, cudaMemcpyHostToDevice, out->stream));
  out->h2d_bytes += (sbytes);
  {
    Prof p(out, "merge", out->geo.n_rec * n);
    merge_kernel<<<grid_blocks(out, out->geo.n_rec, 256, 8), 256, 0, out->stream>>>(
        tmp.as<MergeSrc>(), (uint32_t)n, out->geo.n_rec, now_common, policy == SSPD_UNION_MIN ? 1 : 0,
        out->stamps);
  }
  sspd_status s = check_launch();
  CU(cudaStreamSynchronize(out->stream));
  tmp.release();
  if (s) return s;
  out->now = now_common;
  out->hist_valid = false;
  return SSPD_OK;
}

sspd_status sspd_equal(sspd_grid* a, sspd_grid* b, int* equal) {
  *equal = 0;
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
  int* flag = static_cast<int*>(a->pinned_small);
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
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  if (g->hist) {
    CU(cudaStreamSynchronize(g->stream));
    cudaFree(g->hist);
    g->hist = nullptr;
  }
  g->K = k_max;
  g->hist_valid = false;
  if (k_max) {
    if (cudaMalloc(&g->hist, (size_t)k_max * g->geo.ncells * 4) != cudaSuccess) {
      cudaGetLastError();
      g->K = 0;
      return fail(SSPD_CUDA_ERROR, "CUDA error: out of memory (window ring)");
    }
    return hist_rebuild_locked(g);
  }
  return SSPD_OK;
}

sspd_status sspd_grid_stamps(sspd_grid* g, uint32_t** dev_stamps, uint64_t* words) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  sspd_status s = commit_locked(g);
  if (s) return s;
  CU(cudaStreamSynchronize(g->stream));
  *dev_stamps = g->stamps;
  *words = g->geo.n_rec;
  // the caller may rewrite stamps (e.g. an in-place NCCL max); the ring is
  // rebuilt from them on next use
  g->hist_valid = false;
  return SSPD_OK;
}

sspd_status sspd_grid_touched(sspd_grid* g, uint32_t** dev_bits, uint64_t* words) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
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
  g->profiling = on != 0;
  return SSPD_OK;
}

sspd_status sspd_profile_reset(sspd_grid* g) {
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  cudaStreamSynchronize(g->stream);
  for (auto& r : g->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
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
