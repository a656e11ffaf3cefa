// kernels.cuh -- sm_100a kernels for the sliding super point detector.
//
// Data layout in HBM:
//   stamps  u32[r * 2^q * eta]   (row, column, bucket) order, like the
//                                 reference's cells_ (rsea.hpp:105-112);
//                                 u8/u16 codes on narrow-stamp grids
//   touched u32[ceil(n/32)]      this slot's touched recorders, 1 bit each
//   hist    u32[K * r * 2^q]     per-cell count of buckets whose latest touch
//                                 is slot s, ring-indexed by s mod K (optional)
// A recorder's reference distance is min(now - stamp, 0xFFFF); stamp 0 is
// never-seen and `now` starts at 65535.
//
// Contents, in order: hashing and the pair stream; the scans (bitmap,
// direct, pair-set dedup with the exchange lists) and binning; commit,
// counts and the window ring; hot sets and the reconstruction chain
// (programmatic dependent launches); exact ground truth; conversions, merge
// and equality; sharded routers (own / relay / receive scans, survivor
// masks); narrow stamps.
#pragma once

#include <cstdint>

namespace sspd_dev {

constexpr uint32_t kBaseNow = 65535u;

// Hash tables of HashSeeds (hashing.hpp:41-53), generated on the host with
// the reference seeding (hashing.cpp:8-34).
struct HashTabs {
  uint64_t h1[4][256];
  uint64_t row0[4][256];
};

// Grid geometry as kernel arguments.
struct Geo {
  uint32_t q, r, delta, eta;
  uint32_t col_mask;     // 2^q - 1
  uint32_t low_mask;     // 2^(q-delta) - 1: overlap of adjacent blocks
  uint32_t ncells;       // r * 2^q
  uint64_t n_rec;        // ncells * eta
  // cells [own_lo, own_hi) have stamps on this device: all of them, except
  // on a partial grid of a sharded router (sspd_grid_create_sharded), whose
  // stamp pointer is then based so that cell c's recorders stay at c * eta
  uint32_t own_lo, own_hi;
};

// Window-ring row of a stamp `age` = now - old slots back (1 <= age < K):
// (now - age) mod K from now_slot = now mod K, without a division (a runtime
// `% K` is a MUFU.RCP + fix-up sequence on every first touch).
__device__ __forceinline__ uint32_t ring_back(uint32_t now_slot, uint32_t age, uint32_t K) {
  return now_slot >= age ? now_slot - age : now_slot + K - age;
}

// floor(n / d) for n < 2^40 (recorder indices) and any 32-bit d >= 1:
// shift for powers of two, else a Granlund-Montgomery multiply.
struct Div40 {
  uint64_t magic;
  uint32_t shift;  // total shift for the magic path
  uint32_t pow2;   // 1 => n >> shift
  __host__ static Div40 make(uint32_t d) {
    Div40 v{};
    if ((d & (d - 1)) == 0) {
      v.pow2 = 1;
      v.shift = 0;
      while ((1u << v.shift) < d) ++v.shift;
      v.magic = 0;
    } else {
      uint32_t l = 0;
      while ((1ull << l) < d) ++l;
      v.pow2 = 0;
      v.shift = 40 + l;
      // m = ceil(2^(40+l) / d) < 2^42
      unsigned __int128 num = (unsigned __int128)1 << (40 + l);
      v.magic = (uint64_t)((num + d - 1) / d);
    }
    return v;
  }
  __device__ __forceinline__ uint64_t div(uint64_t n) const {
    if (pow2) return n >> shift;
    return (uint64_t)(((unsigned __int128)n * magic) >> shift);
  }
};

// CHECKED BUILD (-DSSPD_CHECKED, lib/libsspd_cuda_checked.so; compute-
// sanitizer is closed on this pool): every data-dependent index into the
// stamps, narrow codes and window ring is bounds-checked against the grid
// (including a partial grid's own cells), and every window-ring decrement
// asserts the count it takes from is positive -- the ring's invariant.  A
// failed check records the first failing source line and a count in device
// globals (read by sspd_checked_status) and skips the access.  The product
// build compiles all of it away.
#ifdef SSPD_CHECKED
__device__ unsigned int g_chk_line;
__device__ unsigned long long g_chk_count;
__device__ __forceinline__ bool chk_fail(unsigned line) {
  atomicCAS(&g_chk_line, 0u, line);
  atomicAdd(&g_chk_count, 1ull);
  return false;
}
#define SSPD_OK_OR_SKIP(cond) ((cond) ? true : chk_fail(__LINE__))
#else
#define SSPD_OK_OR_SKIP(cond) true
#endif

// Recorder (cell, bucket) of an owned cell.
__device__ __forceinline__ bool rec_ok(const Geo& geo, uint64_t cell, uint32_t bucket) {
  return cell >= geo.own_lo && cell < geo.own_hi && bucket < geo.eta;
}
// Window-ring moves: +1 for the slot now, -1 for the slot a recorder leaves.
__device__ __forceinline__ void ring_add(uint32_t* hist, uint32_t slot, uint32_t ncells, uint32_t cell, uint32_t K,
                                         unsigned line) {
#ifdef SSPD_CHECKED
  if (!(slot < K && cell < ncells)) {
    chk_fail(line);
    return;
  }
#endif
  atomicAdd(hist + (uint64_t)slot * ncells + cell, 1u);
}
__device__ __forceinline__ void ring_sub(uint32_t* hist, uint32_t slot, uint32_t ncells, uint32_t cell, uint32_t K,
                                         unsigned line) {
#ifdef SSPD_CHECKED
  if (!(slot < K && cell < ncells)) {
    chk_fail(line);
    return;
  }
  if (atomicSub(hist + (uint64_t)slot * ncells + cell, 1u) == 0u) chk_fail(line);  // count went below zero
#else
  atomicSub(hist + (uint64_t)slot * ncells + cell, 1u);
#endif
}

// x86 semantics of the reference's 32-bit shifts by computed amounts
// (hashing.hpp:70 can shift by >= 32 for large r): the count is masked.
__device__ __forceinline__ uint32_t shr32(uint32_t x, uint32_t s) { return x >> (s & 31u); }

__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// ---------------------------------------------------------------------------
// SCAN: Rsea::update over a batch (rsea.cpp:29-53).  Three modes, identical
// in result (tests/test_gpu_parity.py runs them all):
//
//  * bitmap (deferred): each touch sets its recorder's bit in the per-slot
//    touched bitmap with red.or; commit_kernel folds the bitmap into the
//    stamps before anything reads them.  When the bitmap fits in L2 (the
//    reference geometry: 20 MiB for 640 MiB of stamps) every touch is an
//    L2-resident atomic and the stamp grid is written once, in address order.
//  * direct: each touch stamps its recorder in place (atomicMax(now) when the
//    window ring is tracked -- the old stamp says which ring entry to move the
//    bucket from -- else red.max).
//  * dedup (scan_dedup_kernel below): direct stamping behind a per-slot set
//    of the (cip, oip) pairs already seen, so a pair repeated within the slot
//    costs one probe instead of r random read-modify-writes.  The default
//    once the grid is far beyond L2 (Zipf traffic repeats pairs heavily).
//
// FILTER: probe the target word through L1 first and skip the atomic when the
// touch is already recorded (bit set / stamp == now).  Both only move one way
// during a scan, so a stale L1 line can cost a redundant atomic but never
// lose one; with Zipf traffic most packets repeat a pair seen this slot.
// H1MODE 0: eta a power of two <= 2^32, H1 needs only its low 32 bits.
// H1MODE 1: general eta, full 64-bit tabulation value % eta (hashing.hpp:58).

struct ScanTables {
  uint16_t row0[4][256];
  uint64_t h1[4][256];  // low 32 bits used in H1MODE 0
};

__device__ __forceinline__ void load_scan_tables(ScanTables& t, const HashTabs* __restrict__ tabs) {
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    t.row0[i >> 8][i & 255] = (uint16_t)tabs->row0[i >> 8][i & 255];
    t.h1[i >> 8][i & 255] = tabs->h1[i >> 8][i & 255];
  }
  __syncthreads();
}

// Row-0 column of cip (rhfg_from_row0's col0, hashing.hpp:68-69).
__device__ __forceinline__ uint32_t row0_col(const ScanTables& t, const Geo& geo, uint32_t cip) {
  return ((uint32_t)t.row0[0][cip & 0xff] ^ t.row0[1][(cip >> 8) & 0xff] ^ t.row0[2][(cip >> 16) & 0xff] ^
          t.row0[3][cip >> 24]) &
         geo.col_mask;
}

// Bucket of oip (hash_opposite, hashing.hpp:56-59).
template <int H1MODE>
__device__ __forceinline__ uint32_t h1_bucket(const ScanTables& t, const Geo& geo, uint32_t oip) {
  if (H1MODE == 0) {
    const uint32_t* lo = reinterpret_cast<const uint32_t*>(&t.h1[0][0]);
    const uint32_t h = lo[2 * (0 * 256 + (oip & 0xff))] ^ lo[2 * (1 * 256 + ((oip >> 8) & 0xff))] ^
                       lo[2 * (2 * 256 + ((oip >> 16) & 0xff))] ^ lo[2 * (3 * 256 + (oip >> 24))];
    return h & (geo.eta - 1u);
  }
  const uint64_t h = t.h1[0][oip & 0xff] ^ t.h1[1][(oip >> 8) & 0xff] ^ t.h1[2][(oip >> 16) & 0xff] ^
                     t.h1[3][oip >> 24];
  return (uint32_t)(h % geo.eta);
}

// Bucket of oip and row-0 column of cip (rsea.cpp:31-32).
template <int H1MODE>
__device__ __forceinline__ void hash_pair(const ScanTables& t, const Geo& geo, uint32_t cip, uint32_t oip,
                                          uint32_t& bucket, uint32_t& col0) {
  bucket = h1_bucket<H1MODE>(t, geo, oip);
  col0 = row0_col(t, geo, cip);
}

// Column of row `row` (rhfg_from_row0, hashing.hpp:68-71).
__device__ __forceinline__ uint32_t row_col(const Geo& geo, uint32_t row, uint32_t cip, uint32_t col0) {
  return row == 0 ? col0 : (shr32(cip, (row - 1) * geo.delta) ^ col0) & geo.col_mask;
}

// Stream the pairs: two pairs per 16-byte load, two loads in flight.
template <class F>
__device__ __forceinline__ void for_each_pair(const uint32_t* __restrict__ pairs, uint64_t n, F&& f) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(pairs) & 15u) == 0) {
    const uint64_t nquads = n >> 1;
    uint64_t i = tid;
    for (; i + nthreads < nquads; i += 2 * nthreads) {
      const uint4 a = ld_stream_u4(pairs + 4 * i);
      const uint4 b = ld_stream_u4(pairs + 4 * (i + nthreads));
      f(a.x, a.y);
      f(a.z, a.w);
      f(b.x, b.y);
      f(b.z, b.w);
    }
    for (; i < nquads; i += nthreads) {
      const uint4 a = ld_stream_u4(pairs + 4 * i);
      f(a.x, a.y);
      f(a.z, a.w);
    }
    if ((n & 1) && tid == 0) f(pairs[2 * (n - 1)], pairs[2 * (n - 1) + 1]);
  } else {
    for (uint64_t i = tid; i < n; i += nthreads) f(pairs[2 * i], pairs[2 * i + 1]);
  }
}

template <int H1MODE, int FILTER>
__global__ void __launch_bounds__(256) scan_bitmap_kernel(const uint32_t* __restrict__ pairs,
                                                          uint64_t n, const HashTabs* __restrict__ tabs,
                                                          Geo geo, uint32_t* __restrict__ touched) {
  __shared__ ScanTables t;
  load_scan_tables(t, tabs);
  for_each_pair(pairs, n, [&](uint32_t cip, uint32_t oip) {
    uint32_t bucket, col0;
    hash_pair<H1MODE>(t, geo, cip, oip, bucket, col0);
    // rows in groups of 4: the L1 probes of a group are issued together
    for (uint32_t r0 = 0; r0 < geo.r; r0 += 4) {
      uint64_t w[4];
      uint32_t bit[4], cur[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t row = r0 + u;
        const uint64_t idx = ((uint64_t)row << geo.q | row_col(geo, row, cip, col0)) * geo.eta + bucket;
        w[u] = idx >> 5;
        bit[u] = 1u << (idx & 31);
        cur[u] = (row < geo.r) ? (FILTER ? __ldca(touched + w[u]) : 0u) : bit[u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (!(cur[u] & bit[u])) red_or(touched + w[u], bit[u]);
    }
  });
}

// HIST: maintain the window ring (K slots) from the old stamps.
// BITS: also record touches in the bitmap (the union-min exchange of a
//       multi-router slot, paper_1803_11036_b200/dist.py).
template <int H1MODE, int FILTER, int HIST, int BITS>
__global__ void __launch_bounds__(256) scan_direct_kernel(const uint32_t* __restrict__ pairs, uint64_t n,
                                                          const HashTabs* __restrict__ tabs, Geo geo,
                                                          uint32_t* __restrict__ stamps, uint32_t now,
                                                          uint32_t* __restrict__ hist, uint32_t K,
                                                          uint32_t* __restrict__ touched) {
  __shared__ ScanTables t;
  load_scan_tables(t, tabs);
  const uint32_t now_slot = HIST ? now % K : 0;
  for_each_pair(pairs, n, [&](uint32_t cip, uint32_t oip) {
    uint32_t bucket, col0;
    hash_pair<H1MODE>(t, geo, cip, oip, bucket, col0);
    for (uint32_t r0 = 0; r0 < geo.r; r0 += 4) {
      uint64_t idx[4];
      uint32_t cell[4], cur[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t row = r0 + u;
        cell[u] = row << geo.q | row_col(geo, row, cip, col0);
        idx[u] = (uint64_t)cell[u] * geo.eta + bucket;
        const bool live = row < geo.r && SSPD_OK_OR_SKIP(rec_ok(geo, cell[u], bucket));
        cur[u] = live ? (FILTER ? __ldca(stamps + idx[u]) : 0u) : now;
      }
      uint32_t old[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // issue the group's atomics before consuming any old value
        old[u] = now;
        if (cur[u] == now) continue;
        if (HIST) old[u] = atomicMax(stamps + idx[u], now);
        else asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(stamps + idx[u]), "r"(now) : "memory");
        if (BITS) red_or(touched + (idx[u] >> 5), 1u << (idx[u] & 31));
      }
      if (HIST) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (old[u] >= now) continue;
          ring_add(hist, now_slot, geo.ncells, cell[u], K, __LINE__);
          if (old[u] + K > now)
            ring_sub(hist, ring_back(now_slot, now - old[u], K), geo.ncells, cell[u], K, __LINE__);
        }
      }
    }
  });
}

// DEDUP (direct stamping behind a per-slot pair set): a pair that repeats
// within the slot touches the same r recorders again, so only the first
// occurrence needs the random-access work.  The set is an open-addressed
// table of exact 64-bit (cip, oip) keys sized to stay L2-resident; a probe
// reads through L1 first (hot pairs hit there once inserted), and insertion
// is an atomicCAS.  Every miss path -- probe limit reached, table full, the
// one key equal to the empty marker -- falls back to "new pair", which is
// only ever redundant work, never a lost touch.  New pairs stamp their r
// recorders like scan_direct_kernel.
constexpr uint64_t kEmptyKey = ~0ull;
#ifndef SSPD_PROBE_LIMIT
#define SSPD_PROBE_LIMIT 8
#endif
constexpr int kProbeLimit = SSPD_PROBE_LIMIT;

// The pair set is split into kPairBins regions; a key's region is the top
// bits of its hash and its slot within the region the low bits, with linear
// probing inside the region.  Binned scans (bin_count/bin_scatter below)
// process the pairs region by region, so the active part of the set stays
// in L2.
constexpr int kPairBinBits = 6;
constexpr int kPairBins = 1 << kPairBinBits;

// A hash of the whole key (exact ground-truth sets).
__device__ __forceinline__ uint64_t pair_mix_hash(uint64_t key) {
  uint64_t h = key * 0x9e3779b97f4a7c15ull;
  return h ^ (h >> 29);
}

// Slot hash of the per-slot pair sets.  SSPD_PAIR_GROUP: every bit but the
// low 4 from the cip alone, the low 4 from the oip, so a host's pairs share
// one 16-slot (128 B) line of the set -- the Zipf head's ~3M repeating pairs
// then live in ~0.2M L2 lines instead of ~3M (one tag each) among the tail's.
#ifndef SSPD_PAIR_GROUP
#define SSPD_PAIR_GROUP 0
#endif
__device__ __forceinline__ uint64_t pair_slot_hash(uint64_t key) {
  if (SSPD_PAIR_GROUP) {
    uint64_t z = (key >> 32) + 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return (z & ~15ull) | ((uint32_t)key * 0x9E3779B1u >> 28);
  }
  return pair_mix_hash(key);
}

__device__ __forceinline__ uint32_t pair_bin(uint64_t h) { return (uint32_t)(h >> (64 - kPairBinBits)); }

// slot of probe i: region base | ((h + i) & region mask); mask = entries - 1
__device__ __forceinline__ uint64_t pair_slot(uint64_t h, int i, uint64_t mask) {
  const uint64_t region_mask = mask >> kPairBinBits;
  return ((uint64_t)pair_bin(h) * (region_mask + 1)) | ((h + i) & region_mask);
}

// Resolve a probe that started with value `v` at probe distance 0.
__device__ __forceinline__ bool pair_resolve(unsigned long long* __restrict__ table, uint64_t mask, uint64_t key,
                                             uint64_t h, unsigned long long v) {
  if (key == kEmptyKey) return true;
  for (int i = 0;; ) {
    const uint64_t slot = pair_slot(h, i, mask);
    if (v == key) return false;
    if (v == kEmptyKey) {
      const unsigned long long old = atomicCAS(table + slot, kEmptyKey, key);
      if (old == kEmptyKey) return true;
      if (old == key) return false;
    }
    if (++i >= kProbeLimit) return true;
    v = __ldca(table + pair_slot(h, i, mask));
  }
}

// Stamp the r recorders of a new pair (direct, with the window ring).
template <int H1MODE, int HIST, int BITS>
__device__ __forceinline__ void stamp_pair(const ScanTables& t, const Geo& geo, uint32_t cip, uint32_t oip,
                                           uint32_t* __restrict__ stamps, uint32_t now, uint32_t now_slot,
                                           uint32_t* __restrict__ hist, uint32_t K, uint32_t* __restrict__ touched) {
  uint32_t bucket, col0;
  hash_pair<H1MODE>(t, geo, cip, oip, bucket, col0);
  for (uint32_t r0 = 0; r0 < geo.r; r0 += 4) {
    uint32_t cell[4], old[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // the atomics of a group are independent: issue them together
      const uint32_t row = r0 + u;
      cell[u] = row << geo.q | row_col(geo, row, cip, col0);
      old[u] = now;
      if (row < geo.r && SSPD_OK_OR_SKIP(rec_ok(geo, cell[u], bucket))) {
        uint32_t* p = stamps + (uint64_t)cell[u] * geo.eta + bucket;
        if (HIST) old[u] = atomicMax(p, now);
        else asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(now) : "memory");
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (r0 + u >= geo.r) break;
      const uint64_t idx = (uint64_t)cell[u] * geo.eta + bucket;
      if (HIST && old[u] < now) {
        ring_add(hist, now_slot, geo.ncells, cell[u], K, __LINE__);
        if (old[u] + K > now) ring_sub(hist, ring_back(now_slot, now - old[u], K), geo.ncells, cell[u], K, __LINE__);
      }
      if (BITS) red_or(touched + (idx >> 5), 1u << (idx & 31));
    }
  }
}

// EXPORT: append each new pair to `out_pairs` (the slot's distinct pairs,
// exchanged between routers instead of a bitmap; paper_1803_11036_b200/dist.py).
// PUSH (with EXPORT): also store each new pair, at the same position, into
// every peer router's inbox region for this router -- P2P stores over NVLink
// into symmetric memory, so the exchange overlaps the scan instead of
// following it.  `peers[p]` is router p's inbox (base of world regions of
// `region_cap` pairs); positions past region_cap are dropped and the host
// falls back to an all-gather for that slot.
// Each thread takes 4 pairs per iteration and issues their 4 first probes
// together before resolving any (the probes are the latency chain).
// Append-only pair lists (the exchange list, peer inboxes) grown in blocks:
// a warp reserves kListBlock slots with ONE atomic and fills them over
// several iterations, instead of one atomic per warp per iteration on a
// counter every warp of the GPU shares (that contention cost 13 vs 3.5 ms
// per C2 slot, profiles/r01_ab_list_blocks.md).  The warp's last block is
// padded with copies of its last pair, so a list is dense up to its counter;
// a repeated pair is harmless to every consumer (stamping is idempotent).
constexpr uint32_t kListBlock = 64;

struct ListState {
  unsigned long long base;  // first slot of the warp's current block
  uint32_t fill;            // slots used in it (kListBlock: no block yet)
  uint32_t unused;
  uint2 last;               // the last pair appended (the padding value)
};

__device__ __forceinline__ void list_init(ListState& st, uint32_t lane) {
  if (lane == 0) {
    st.base = 0;
    st.fill = kListBlock;
  }
  __syncwarp();
}

// The lanes of `m` with `mine` set append `pr`; returns this lane's slot
// (meaningful only when `mine`).  Call with the same `m` on every lane in it.
__device__ __forceinline__ uint64_t list_append(ListState& st, unsigned long long* counter, unsigned m, bool mine,
                                                uint2 pr, uint32_t lane) {
  const unsigned b = __ballot_sync(m, mine);
  if (!b) return 0;
  const uint32_t cnt = __popc(b), rank = __popc(b & ((1u << lane) - 1u));
  const int leader = __ffs(m) - 1;
  const uint32_t fill = st.fill;
  const unsigned long long base = st.base;
  const uint32_t room = kListBlock - fill;
  unsigned long long nb = 0;
  if (cnt > room) {
    if ((int)lane == leader) nb = atomicAdd(counter, (unsigned long long)kListBlock);
    nb = __shfl_sync(m, nb, leader);
  }
  const uint64_t pos = rank < room ? base + fill + rank : nb + (rank - room);
  __syncwarp(m);
  if ((int)lane == leader) {
    if (cnt > room) {
      st.base = nb;
      st.fill = cnt - room;
    } else {
      st.fill = fill + cnt;
    }
  }
  if ((int)lane == 31 - __clz(b)) st.last = pr;
  __syncwarp(m);
  return pos;
}

// After the loop (all 32 lanes): the unused tail of the warp's block, padded.
template <class W>
__device__ __forceinline__ void list_pad(ListState& st, uint32_t lane, W&& write) {
  __syncwarp();
  const uint32_t fill = st.fill;
  for (uint32_t i = fill + lane; i < kListBlock; i += 32) write(st.base + i, st.last);
}

struct PushArgs {
  uint2* const* peers;  // device array of `world` inbox pointers (peer-mapped)
  uint32_t world, rank;
  uint64_t region_cap;
};

// Tuned on B200 at C2 (profiles/r01_ab_dedup_tuning*.txt): 2 pairs per
// thread with every fresh pair's stamp atomics issued before any old value
// is consumed beat 4 pairs with per-pair round trips (3.64 vs 3.76 ms/slot);
// 8 pairs or tighter register caps were slower.
#ifndef SSPD_DEDUP_PPT
#define SSPD_DEDUP_PPT 2  // pairs per thread per iteration (probes in flight)
#endif
#ifndef SSPD_DEDUP_MINB
#define SSPD_DEDUP_MINB 1
#endif
#ifndef SSPD_DEDUP_BATCH_ATOMICS
#define SSPD_DEDUP_BATCH_ATOMICS 1
#endif

template <int H1MODE, int HIST, int BITS, int EXPORT, int PUSH = 0>
__global__ void __launch_bounds__(256, SSPD_DEDUP_MINB) scan_dedup_kernel(const uint32_t* __restrict__ pairs, uint64_t n,
                                                         const HashTabs* __restrict__ tabs, Geo geo,
                                                         unsigned long long* __restrict__ table,
                                                         uint64_t table_mask, uint32_t* __restrict__ stamps,
                                                         uint32_t now, uint32_t* __restrict__ hist, uint32_t K,
                                                         uint32_t* __restrict__ touched,
                                                         uint2* __restrict__ out_pairs,
                                                         unsigned long long* __restrict__ out_count,
                                                         PushArgs push = PushArgs{}) {
  __shared__ ScanTables t;
  __shared__ ListState s_list[8];  // EXPORT: one list state per warp (blockDim 256)
  load_scan_tables(t, tabs);
  const uint32_t now_slot = HIST ? now % K : 0;
  const uint32_t lane = threadIdx.x & 31;
  ListState& wl = s_list[threadIdx.x >> 5];
  if (EXPORT) list_init(wl, lane);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(pairs) & 15u) == 0;
  // group g covers pairs [P g, P g + P): P/2 16-byte loads
  constexpr int P = SSPD_DEDUP_PPT;
  const uint64_t ngroups = (n + P - 1) / P;
  for (uint64_t g = tid; g < ngroups; g += nthreads) {
    uint32_t c[P], o[P];
    bool valid[P];
    const uint64_t p0 = g * P;
    if (vec && p0 + P <= n) {
#pragma unroll
      for (int u = 0; u < P; u += 2) {
        const uint4 a = ld_stream_u4(pairs + 2 * (p0 + u));
        c[u] = a.x; o[u] = a.y; c[u + 1] = a.z; o[u + 1] = a.w;
        valid[u] = valid[u + 1] = true;
      }
    } else {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        valid[u] = p0 + u < n;
        c[u] = valid[u] ? pairs[2 * (p0 + u)] : 0u;
        o[u] = valid[u] ? pairs[2 * (p0 + u) + 1] : 0u;
      }
    }
    uint64_t key[P], h[P];
    unsigned long long v[P];
    bool probe[P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      key[u] = (uint64_t)c[u] << 32 | o[u];
      h[u] = pair_slot_hash(key[u]);
      probe[u] = valid[u];
      v[u] = probe[u] ? __ldca(table + pair_slot(h[u], 0, table_mask)) : 0ull;
    }
    bool fresh[P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      fresh[u] = probe[u] && pair_resolve(table, table_mask, key[u], h[u], v[u]);
    }
    if (EXPORT) {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const unsigned m = __activemask();
        const uint2 pr = make_uint2(c[u], o[u]);
        const uint64_t pos = list_append(wl, out_count, m, fresh[u], pr, lane);
        if (fresh[u]) {
          out_pairs[pos] = pr;
          if (PUSH && pos < push.region_cap)
            for (uint32_t p = 0; p < push.world; ++p)
              if (p != push.rank) push.peers[p][(uint64_t)push.rank * push.region_cap + pos] = pr;
        }
      }
    }
#if SSPD_DEDUP_BATCH_ATOMICS
    // Issue the stamp atomics of every fresh pair of the group before
    // consuming any old value (one exposed round trip per group, not per pair).
    if (HIST && !BITS && geo.r <= 8) {
      uint32_t bucket[P], col0[P], old[P][8];
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (!fresh[u]) continue;
        hash_pair<H1MODE>(t, geo, c[u], o[u], bucket[u], col0[u]);
#pragma unroll
        for (uint32_t row = 0; row < 8; ++row) {
          old[u][row] = now;
          if (row < geo.r &&
              SSPD_OK_OR_SKIP(rec_ok(geo, row << geo.q | row_col(geo, row, c[u], col0[u]), bucket[u])))
            old[u][row] = atomicMax(stamps + (uint64_t)(row << geo.q | row_col(geo, row, c[u], col0[u])) * geo.eta +
                                        bucket[u],
                                    now);
        }
      }
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (!fresh[u]) continue;
#pragma unroll
        for (uint32_t row = 0; row < 8; ++row) {
          if (row >= geo.r || old[u][row] >= now) continue;
          const uint32_t cell = row << geo.q | row_col(geo, row, c[u], col0[u]);
          ring_add(hist, now_slot, geo.ncells, cell, K, __LINE__);
          if (old[u][row] + K > now) ring_sub(hist, ring_back(now_slot, now - old[u][row], K), geo.ncells, cell, K, __LINE__);
        }
      }
      continue;
    }
#endif
#pragma unroll
    for (int u = 0; u < P; ++u)
      if (fresh[u]) stamp_pair<H1MODE, HIST, BITS>(t, geo, c[u], o[u], stamps, now, now_slot, hist, K, touched);
  }
  if (EXPORT)
    list_pad(wl, lane, [&](uint64_t pos, uint2 pr) {
      out_pairs[pos] = pr;
      if (PUSH && pos < push.region_cap)
        for (uint32_t p = 0; p < push.world; ++p)
          if (p != push.rank) push.peers[p][(uint64_t)push.rank * push.region_cap + pos] = pr;
    });
  if (PUSH) __threadfence_system();  // peer stores visible before the exchange's barrier
}

// PIPELINED DEDUP SCAN (the default C2 path: window ring on, no bitmap, no
// exchange list, r <= 8).  Same results as scan_dedup_kernel<.., HIST=1,
// BITS=0, EXPORT=0>; the difference is WHEN each fresh pair's r stamp
// atomics run: a thread's fresh pairs of group i are hashed as soon as their
// probes resolve, and their atomics are issued one iteration later, together
// with group i+1's pair-set probes, so the atomics' round trip is not on the
// critical path of one group:
//   iteration i: load pairs(i) -> probe(i) | atomics(i-1) -> resolve(i)
//                -> ring(i-1) -> hash(i)
// Requesting the recorder lines early (prefetch.global.L2 variants, or a
// cp.async.bulk.prefetch) measured 23-24% SLOWER than none at C2, and an
// L2-resident front set of pairs seen twice (probed first, evict_last) 1.9-2x
// slower: the extra dependent round trip for every pair outweighs the misses
// it saves (profiles/r02_ab_scan.md); nothing is prefetched or fronted.
// HINT 1: L2 eviction priorities -- the random stamp atomics evict_first
// (each stamp line is used once per slot), the pair-set probes
// evict_last (head pairs repeat all slot long), the streamed pairs
// evict_first -- so the stamps' 47M lines per C2 slot do not push the
// pair set's hot lines out of L2.
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint32_t atom_max_hint(uint32_t* p, uint32_t v, uint64_t pol) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.max.L2::cache_hint.u32 %0, [%1], %2, %3;"
               : "=r"(old) : "l"(p), "r"(v), "l"(pol) : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_ca_hint(const unsigned long long* p, uint64_t pol) {
  unsigned long long v;
  asm volatile("ld.global.ca.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u4_hint(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// pair_resolve with the pair-set cache policy on its probes
__device__ __forceinline__ bool pair_resolve_hint(unsigned long long* __restrict__ table, uint64_t mask, uint64_t key,
                                                  uint64_t h, unsigned long long v, uint64_t pol) {
  if (key == kEmptyKey) return true;
  for (int i = 0;;) {
    const uint64_t slot = pair_slot(h, i, mask);
    if (v == key) return false;
    if (v == kEmptyKey) {
      const unsigned long long old = atomicCAS(table + slot, kEmptyKey, key);  // (atom.cas takes no cache hint)
      if (old == kEmptyKey) return true;
      if (old == key) return false;
    }
    if (++i >= kProbeLimit) return true;
    v = ld_ca_hint(table + pair_slot(h, i, mask), pol);
  }
}

// SECTOR PROBES (SSPD_PIPE_SECT): the pair set read 32 B at a time -- the
// 4 slots of the sector holding a key's home slot in ONE 256-bit load
// (LDG.E.ENL2.256) -- so a collision inside the sector costs no dependent
// round trip; sectors are then probed in order, and empty slots are claimed
// in slot order, so concurrent inserters of one key agree.  (Exact: "seen"
// only on a key match; a probe limit reads as fresh.)
struct Sect {
  unsigned long long k[4];
};
__device__ __forceinline__ Sect ld_sect(const unsigned long long* p) {
  Sect s;
  asm volatile("ld.global.ca.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(s.k[0]), "=l"(s.k[1]), "=l"(s.k[2]), "=l"(s.k[3])
               : "l"(p));
  return s;
}
__device__ __forceinline__ uint64_t sect_base(uint64_t h, int i, uint64_t mask) {
  return pair_slot(h & ~3ull, 4 * i, mask);  // region base | ((h & ~3) + 4i) & region mask
}
// SSPD_PIPE_SECT 2 -- HOST GROUPS: a cip's pairs share a 32-slot group (two
// 128 B lines, 8 sectors; group index from the cip alone), a pair's first
// sector from its oip; probes walk the group's sectors.  The Zipf head's
// ~3M repeating pairs then sit in ~0.2M groups (~0.4M L2 lines) instead of
// ~3M lines among the tail's, at one sector load per probe.
__device__ __forceinline__ uint64_t host_group_hash(uint64_t key) {
  uint64_t z = (key >> 32) + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return (z & ~31ull) | ((uint64_t)((uint32_t)key * 0x9E3779B1u >> 29) << 2);
}
__device__ __forceinline__ uint64_t group_sect_base(uint64_t h, int i, uint64_t mask) {
  return (h & ~31ull & mask) | ((((h >> 2) + (uint64_t)i) & 7ull) << 2);
}
constexpr int kSectLimit = 4;
template <int GROUP = 0>
__device__ __forceinline__ bool sect_resolve(unsigned long long* __restrict__ table, uint64_t mask, uint64_t key,
                                             uint64_t h, Sect v) {
  if (key == kEmptyKey) return true;
  for (int i = 0;;) {
    const uint64_t base = GROUP ? group_sect_base(h, i, mask) : sect_base(h, i, mask);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (v.k[j] == key) return false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (v.k[j] != kEmptyKey) continue;
      const unsigned long long old = atomicCAS(table + base + j, kEmptyKey, key);
      if (old == kEmptyKey) return true;
      if (old == key) return false;
    }
    if (++i >= kSectLimit) return true;
    v = ld_sect(table + (GROUP ? group_sect_base(h, i, mask) : sect_base(h, i, mask)));
  }
}

#ifndef SSPD_PIPE_SECT
#define SSPD_PIPE_SECT 0
#endif
// SSPD_PIPE_CPASYNC: each thread copies its NEXT group's pairs (16 B) into its
// own shared-memory slot with cp.async (LDGSTS) while it works on the current
// one, so the pair stream's DRAM latency leaves the per-iteration chain
// without holding registers; warp-private double buffer, no CTA barrier.
#ifndef SSPD_PIPE_CPASYNC
#define SSPD_PIPE_CPASYNC 0
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// SSPD_PIPE_LDPF: load (not prefetch) each fresh pair's recorders when it is
// hashed, so its deferred atomics hit L2 (the ld-then-atomic pattern
// tools/fetch_probe.cu measured fastest; prefetch.global.L2 measured slow):
// 1 = loads whose values are never read, 2 = values carried to the next
// iteration and folded into a sink before the atomics.
#ifndef SSPD_PIPE_LDPF
#define SSPD_PIPE_LDPF 0
#endif
__device__ __forceinline__ uint32_t ld_cg_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// R: rows at compile time (5, the reference default), or 0 = geo.r <= 8.
#ifndef SSPD_PIPE_MINB
#define SSPD_PIPE_MINB 4
#endif
#ifndef SSPD_PIPE_PPT
#define SSPD_PIPE_PPT 2  // pairs per thread per iteration (1, 2 or 4)
#endif
template <int H1MODE, int HINT, int R>
__global__ void __launch_bounds__(256, SSPD_PIPE_MINB) scan_dedup_pipe_kernel(
    const uint32_t* __restrict__ pairs, uint64_t n, const HashTabs* __restrict__ tabs, Geo geo,
    unsigned long long* __restrict__ table, uint64_t table_mask, uint32_t* __restrict__ stamps, uint32_t now,
    uint32_t* __restrict__ hist, uint32_t K, unsigned long long* __restrict__ fresh_count) {
  __shared__ ScanTables t;
  load_scan_tables(t, tabs);
  const uint32_t now_slot = now % K;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(pairs) & 15u) == 0;
  const uint64_t pol_stamp = HINT ? l2_policy_first() : 0, pol_set = HINT ? l2_policy_last() : 0;
  constexpr int P = SSPD_PIPE_PPT;
  constexpr uint32_t RM = R ? R : 8;  // unrolled row count
  const uint32_t nr = R ? R : geo.r;
  const uint64_t ngroups = (n + P - 1) / P;
  uint32_t n_fresh = 0;
  // the previous group's fresh pairs: cip, bucket, row-0 column
  uint32_t pc[P], pb[P], p0[P];
  bool pv[P];
  uint32_t ldv[SSPD_PIPE_LDPF == 2 ? P : 1][SSPD_PIPE_LDPF == 2 ? RM : 1];
  uint32_t sink = 0;
#pragma unroll
  for (int u = 0; u < P; ++u) pv[u] = false;
  // one extra round per thread drains the last group's pending stamps
  constexpr bool kCp = SSPD_PIPE_CPASYNC && P == 2;
  __shared__ uint4 s_next[kCp ? 2 : 1][kCp ? 256 : 1];
  auto full_group = [&](uint64_t gg) { return gg < ngroups && vec && gg * P + P <= n; };
  if (kCp) {
    if (full_group(tid)) cp_async16(&s_next[0][threadIdx.x], pairs + 2 * (tid * P));
    cp_async_commit();
  }
  uint32_t it = 0;
  for (uint64_t g = tid; g < ngroups + nthreads; g += nthreads, ++it) {
    const bool have = g < ngroups;
    uint32_t c[P], o[P];
    bool valid[P];
    const uint64_t q0 = g * P;
    if (kCp) {
      // queue the next group's copy, then wait for this one's
      if (full_group(g + nthreads))
        cp_async16(&s_next[(it + 1) & 1][threadIdx.x], pairs + 2 * ((g + nthreads) * P));
      cp_async_commit();
      cp_async_wait<1>();
    }
    if (kCp && full_group(g)) {
      const uint4 a = s_next[it & 1][threadIdx.x];
      c[0] = a.x; o[0] = a.y; c[P - 1] = a.z; o[P - 1] = a.w;
      valid[0] = valid[P - 1] = true;
    } else if (P >= 2 && have && vec && q0 + P <= n) {
#pragma unroll
      for (int u = 0; u < P; u += 2) {
        const uint4 a = HINT ? ld_stream_u4_hint(pairs + 2 * (q0 + u), pol_stamp) : ld_stream_u4(pairs + 2 * (q0 + u));
        c[u] = a.x; o[u] = a.y; c[u + 1] = a.z; o[u + 1] = a.w;
        valid[u] = valid[u + 1] = true;
      }
    } else {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        valid[u] = have && q0 + u < n;
        c[u] = valid[u] ? pairs[2 * (q0 + u)] : 0u;
        o[u] = valid[u] ? pairs[2 * (q0 + u) + 1] : 0u;
      }
    }
    uint64_t key[P], h[P];
    unsigned long long v[P];
    Sect sv[SSPD_PIPE_SECT ? P : 1];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      key[u] = (uint64_t)c[u] << 32 | o[u];
      h[u] = SSPD_PIPE_SECT == 2 ? host_group_hash(key[u]) : pair_slot_hash(key[u]);
      if (SSPD_PIPE_SECT) {
        if (valid[u])
          sv[u] = ld_sect(table + (SSPD_PIPE_SECT == 2 ? group_sect_base(h[u], 0, table_mask)
                                                       : sect_base(h[u], 0, table_mask)));
        v[u] = 0ull;
      } else {
        unsigned long long* slot0 = table + pair_slot(h[u], 0, table_mask);
        v[u] = valid[u] ? (HINT ? ld_ca_hint(slot0, pol_set) : __ldca(slot0)) : 0ull;
      }
    }
    // the previous group's stamps, in flight together with this group's probes
    uint32_t old[P][RM];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (!pv[u]) continue;
      if (SSPD_PIPE_LDPF == 2)
#pragma unroll
        for (uint32_t row = 0; row < RM; ++row)
          if (row < nr) sink ^= ldv[SSPD_PIPE_LDPF == 2 ? u : 0][SSPD_PIPE_LDPF == 2 ? row : 0];
#pragma unroll
      for (uint32_t row = 0; row < RM; ++row)
        if (row < nr) {
          const uint32_t cell = row << geo.q | row_col(geo, row, pc[u], p0[u]);
          uint32_t* sp = stamps + (uint64_t)cell * geo.eta + pb[u];
          old[u][row] = now;
          if (SSPD_OK_OR_SKIP(rec_ok(geo, cell, pb[u])))
            old[u][row] = HINT ? atom_max_hint(sp, now, pol_stamp) : atomicMax(sp, now);
        }
    }
    bool fresh[P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (SSPD_PIPE_SECT)
        fresh[u] = valid[u] && sect_resolve<SSPD_PIPE_SECT == 2>(table, table_mask, key[u], h[u],
                                                                 sv[SSPD_PIPE_SECT ? u : 0]);
      else
        fresh[u] = valid[u] && (HINT ? pair_resolve_hint(table, table_mask, key[u], h[u], v[u], pol_set)
                                     : pair_resolve(table, table_mask, key[u], h[u], v[u]));
    }
    // window ring moves for the previous group's first touches
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (!pv[u]) continue;
#pragma unroll
      for (uint32_t row = 0; row < RM; ++row) {
        if (row >= nr || old[u][row] >= now) continue;
        const uint32_t cell = row << geo.q | row_col(geo, row, pc[u], p0[u]);
        ring_add(hist, now_slot, geo.ncells, cell, K, __LINE__);
        if (old[u][row] + K > now)
          ring_sub(hist, ring_back(now_slot, now - old[u][row], K), geo.ncells, cell, K, __LINE__);
      }
    }
    // this group's fresh pairs become pending
#pragma unroll
    for (int u = 0; u < P; ++u) {
      pv[u] = fresh[u];
      n_fresh += fresh[u];
      if (!fresh[u]) continue;
      pc[u] = c[u];
      hash_pair<H1MODE>(t, geo, c[u], o[u], pb[u], p0[u]);
      if (SSPD_PIPE_LDPF)
#pragma unroll
        for (uint32_t row = 0; row < RM; ++row)
          if (row < nr) {
            const uint32_t v = ld_cg_volatile(stamps + (uint64_t)(row << geo.q | row_col(geo, row, pc[u], p0[u])) *
                                                           geo.eta + pb[u]);
            if (SSPD_PIPE_LDPF == 2) ldv[SSPD_PIPE_LDPF == 2 ? u : 0][SSPD_PIPE_LDPF == 2 ? row : 0] = v;
          }
    }
  }
  if (SSPD_PIPE_LDPF == 2 && sink == 0x9e3779b9u && now == 0u && fresh_count) *fresh_count = sink;  // keep the loads
  // pairs new to this slot (pair-set inserts plus probe-limit misses): one
  // atomic per warp
  if (fresh_count) {
#pragma unroll
    for (int off = 16; off; off >>= 1) n_fresh += __shfl_xor_sync(0xffffffffu, n_fresh, off);
    if ((threadIdx.x & 31) == 0 && n_fresh) atomicAdd(fresh_count, (unsigned long long)n_fresh);
  }
}

// COMPACT KEY SET SCAN (the default C2 path when eta <= 2^16: window ring
// on, no bitmap, no exchange list, r <= 8).  Same results as the pipelined
// dedup scan above; what changes is the per-slot set.
//  * The key is (cip, bucket(oip)), not (cip, oip): the r recorders a pair
//    stamps are (row, col_row(cip), bucket) (rsea.cpp:31-36), so two pairs
//    with one key stamp the same recorders and the second is redundant.
//    With eta <= 2^16 the key has 48 bits.
//  * x = perm48(key) is a bijection of 48-bit values.  Its top bits pick
//    the key's home bucket (BW = 4 u32 entries, one 16 B load; BUCKETS
//    below); the remaining rb bits (the remainder) are stored with the
//    bucket displacement d: entry = (d + 1) << rb | remainder, 0 = empty.
//    An entry in bucket b therefore names exactly one key (home b - d,
//    remainder), so a match is exact: "seen" is never wrong, and every miss
//    path (the walk limit) reads as fresh, which only costs redundant stamps.
//  * 4 B per entry instead of 8: at 2^24 entries the table is 64 MiB, and
//    the ~9.4M keys of a C2 slot load it to 0.56.  On its own such a table
//    is served from L2 (random 16 B probes run at the L2 rate up to 96 MiB,
//    profiles/r02_l2_probe.txt); beside the slot's 47M stamp atomics about
//    half its probe sectors still miss, against ~52M misses per 100M probes
//    for the 256 MiB table of 8-byte keys (profiles/r02_ab_keyset.md).
// Concurrent inserters of one key walk the same slots and compare the same
// expected entry: one CAS wins, the others read it back as "seen".
// BW = 1 (linear probing by slot, entry = (d + 1) << 24 | remainder) and
// BW = 8 remain as compile-time A/B variants (SSPD_CSET_BW).
// A/B diagnostics of the key-set scan's cost split (never the product build;
// their results are wrong): 1 = no window-ring moves (the stamps compile to non-returning
// reds), 2 = non-returning red.max stamps without a cache hint, 3 = returning stamps, no ring moves
#ifndef SSPD_AB_DIAG
#define SSPD_AB_DIAG 0
#endif
#ifndef SSPD_CSET_PROBE_LIMIT
#define SSPD_CSET_PROBE_LIMIT 32
#endif
#ifndef SSPD_CSET_PF
#define SSPD_CSET_PF 0
#endif
#ifndef SSPD_CSET_BW
#define SSPD_CSET_BW 4  // entries per probe bucket: 1 (linear probing by slot), 4 or 8
#endif
constexpr uint32_t kCsetMinLog2 = 24, kCsetMaxLog2 = 30;
// first size 2^24 (64 MiB); the host grows it while a slot's keys load it
// past kCsetMaxLoad, and shrinks it again below kCsetMinLoad (sspd_cuda.cu
// cset_slot_end_locked).  With 4-entry
// buckets the smallest set that holds the keys is the fastest (C2: 2^24 at
// load 0.56 beat 2^25 and 2^26; C2 with 64-entry pools: 2^24 at 0.92 still
// beat 2^25, profiles/r02_ab_keyset.md), so growth only keeps the table
// clear of the overflow cliff.
constexpr uint32_t kCsetStartLog2 = 24;
constexpr double kCsetMaxLoad = 0.75;
constexpr double kCsetMinLoad = 0.15;  // below it the host halves the set (never under kCsetStartLog2)

#ifndef SSPD_CSET_PERM
#define SSPD_CSET_PERM 0  // 1: one odd multiply (Fibonacci hashing: the home is the product's top bits)
#endif
__device__ __forceinline__ uint64_t cset_perm48(uint64_t x) {
  constexpr uint64_t M = (1ull << 48) - 1;
  if (SSPD_CSET_PERM == 1) return (x * 0x9E3779B97F4Bull) & M;
  x = (x * 0x9E3779B97F4Bull) & M;  // odd multipliers and xor-shifts: each step is invertible mod 2^48
  x ^= x >> 23;
  x = (x * 0xC2B2AE3D27D5ull) & M;
  x ^= x >> 25;
  x = (x * 0x165667B19E37ull) & M;
  x ^= x >> 24;
  return x;
}

__device__ __forceinline__ bool cset_resolve(uint32_t* __restrict__ table, uint32_t mask, uint32_t home,
                                             uint32_t rem, uint32_t v) {
  for (uint32_t d = 0;;) {
    const uint32_t want = (d + 1) << 24 | rem;
    if (v == want) return false;
    if (v == 0u) {
      const uint32_t old = atomicCAS(table + ((home + d) & mask), 0u, want);
      if (old == 0u) return true;
      if (old == want) return false;
    }
    if (++d >= SSPD_CSET_PROBE_LIMIT) return true;
    v = __ldca(table + ((home + d) & mask));
  }
}

__device__ __forceinline__ uint32_t ld_ca_hint_u32(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.ca.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// BUCKETS (BW = 4 or 8 entries, one 16 B / 32 B load): the home is a
// bucket, a key sits anywhere in it (empties claimed in slot order), and a
// full bucket overflows into the next.  One load resolves nearly every probe
// (at load 0.28, P(more than 4 keys in a 4-entry bucket) < 1%), so a warp no
// longer waits for its longest linear-probe chain.  The entry stores the
// bucket displacement: entry = (d + 1) << rb | remainder, with rb = 48 -
// log2(buckets) remainder bits.
// Linear runs of full buckets have a long tail: at load 0.56 a sequential
// insert of 9.4M keys displaces a few hundred keys past 8 buckets, none past
// 17; at 0.75 none past 53 (2^24 entries).  48 fits the displacement field at
// every size (lg >= 24: 32 - rb >= 6 bits) and only the rare long run walks it.
constexpr uint32_t kCsetBucketLimit = 48;
template <int BW>
struct CBucket {
  uint32_t e[BW];
};
template <int BW, int HINT>
__device__ __forceinline__ CBucket<BW> ld_bucket(const uint32_t* p, uint64_t pol) {
  CBucket<BW> b;
  if (BW == 4) {
    if (HINT)
      asm volatile("ld.global.ca.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=r"(b.e[0]), "=r"(b.e[1]), "=r"(b.e[2]), "=r"(b.e[3]) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.ca.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b.e[0]), "=r"(b.e[1]), "=r"(b.e[2]), "=r"(b.e[3]) : "l"(p));
  } else {
    uint64_t w[4];
    if (HINT)
      asm volatile("ld.global.ca.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                   : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p), "l"(pol));
    else
      asm volatile("ld.global.ca.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      b.e[2 * j] = (uint32_t)w[j];
      b.e[2 * j + 1] = (uint32_t)(w[j] >> 32);
    }
  }
  return b;
}
// Buckets d >= 1 of a probe, out of line: a 48-bucket walk inlined into the
// probe loop cost the common one-bucket probe 35% at C2 (4.32 vs 3.19 ms),
// and an 8-bucket inline walk overflowed a few hundred keys per slot.  The
// call costs one spilled register in the probe loop (ptxas: 8 B; the SASS
// has one STL and one LDL per iteration, which hit L1).  Even so this is
// 1.5% faster at C2 than a spill-free two-stage inline walk
// (profiles/r02_ab_keyset.md A/B 4; that variant was removed).
template <int BW, int HINT>
__device__ __noinline__ bool cset_resolve_far(uint32_t* __restrict__ table, uint32_t bmask, uint32_t hb,
                                              uint32_t rem, uint32_t rb, uint64_t pol) {
  for (uint32_t d = 1; d < kCsetBucketLimit; ++d) {
    const CBucket<BW> v = ld_bucket<BW, HINT>(table + (uint64_t)((hb + d) & bmask) * BW, pol);
    const uint32_t want = (d + 1) << rb | rem;
    uint32_t* base = table + (uint64_t)((hb + d) & bmask) * BW;
#pragma unroll
    for (int j = 0; j < BW; ++j)
      if (v.e[j] == want) return false;
#pragma unroll
    for (int j = 0; j < BW; ++j) {
      if (v.e[j] != 0u) continue;
      const uint32_t old = atomicCAS(base + j, 0u, want);
      if (old == 0u) return true;
      if (old == want) return false;
    }
  }
  return true;
}

template <int BW, int HINT>
__device__ __forceinline__ bool cset_resolve_bucket(uint32_t* __restrict__ table, uint32_t bmask, uint32_t hb,
                                                    uint32_t rem, uint32_t rb, CBucket<BW> v, uint64_t pol) {
  const uint32_t want = 1u << rb | rem;  // displacement 0: the home bucket, already loaded
  uint32_t* base = table + (uint64_t)hb * BW;
#pragma unroll
  for (int j = 0; j < BW; ++j)
    if (v.e[j] == want) return false;
#pragma unroll
  for (int j = 0; j < BW; ++j) {
    if (v.e[j] != 0u) continue;
    const uint32_t old = atomicCAS(base + j, 0u, want);
    if (old == 0u) return true;
    if (old == want) return false;
  }
  return cset_resolve_far<BW, HINT>(table, bmask, hb, rem, rb, pol);
}

// Narrow-stamp touch and ring helpers (see NARROW STAMPS below); here so
// that the key-set scan can run on 16-bit grids too.
struct NarrowCodes {
  uint32_t now;     // code(now)
  uint32_t lo;      // smallest live code
};

__device__ __forceinline__ uint32_t narrow_max(uint16_t* p, uint32_t code) {
  uint32_t* w = reinterpret_cast<uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
  const bool upper = (reinterpret_cast<uintptr_t>(p) & 2u) != 0;
  const unsigned short a = upper ? 0 : (unsigned short)code, b = upper ? (unsigned short)code : 0;
  unsigned short oa, ob;
  asm volatile("atom.global.max.noftz.v2.bf16 {%0, %1}, [%2], {%3, %4};"
               : "=h"(oa), "=h"(ob)
               : "l"(w), "h"(a), "h"(b)
               : "memory");
  return upper ? ob : oa;
}

// u8: CAS on the containing word, starting from the value `cur` read earlier.
__device__ __forceinline__ uint32_t narrow_max_from(uint8_t* p, uint32_t code, uint32_t cur) {
  uint32_t* w = reinterpret_cast<uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3));
  const uint32_t sh = (uint32_t)(reinterpret_cast<uintptr_t>(p) & 3u) * 8u;
  for (;;) {
    const uint32_t old = (cur >> sh) & 0xffu;
    if (old >= code) return old;
    const uint32_t prev = atomicCAS(w, cur, (cur & ~(0xffu << sh)) | (code << sh));
    if (prev == cur) return old;
    cur = prev;
  }
}

__device__ __forceinline__ uint32_t word_of(const uint8_t* p) {
  return __ldcg(reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(3)));
}

// Ring bookkeeping of one touch whose previous code was `old`.
__device__ __forceinline__ void narrow_ring(uint32_t old, uint32_t cell, const NarrowCodes& nc, uint32_t now,
                                           uint32_t now_slot, const Geo& geo, uint32_t* __restrict__ hist,
                                           uint32_t K) {
  if (old >= nc.now) return;  // already stamped this slot
  ring_add(hist, now_slot, geo.ncells, cell, K, __LINE__);
  if (old >= nc.lo) {
    const uint32_t age = nc.now - old;
    if (age < K) ring_sub(hist, ring_back(now_slot, age, K), geo.ncells, cell, K, __LINE__);
  }
}

// Pipelined exactly like scan_dedup_pipe_kernel: iteration i loads and
// probes group i while group i-1's stamp atomics are in flight.
// HINT 1: the set's probes evict_last, the stamps and the pair stream
// evict_first.
// CT = uint16_t: a 16-bit grid (NARROW STAMPS), each touch one packed-bf16
// max atomic of code(now) = nc.now and the ring moved by narrow_ring.
template <int H1MODE, int HINT, int R, int BW, class CT = uint32_t>
__global__ void __launch_bounds__(256, SSPD_PIPE_MINB) scan_cset_kernel(
    const uint32_t* __restrict__ pairs, uint64_t n, const HashTabs* __restrict__ tabs, Geo geo,
    uint32_t* __restrict__ table, uint32_t lg, CT* __restrict__ stamps, uint32_t now,
    uint32_t* __restrict__ hist, uint32_t K, unsigned long long* __restrict__ fresh_count, uint32_t part = 0,
    uint32_t part_shift = 31, NarrowCodes nc = {}) {
  constexpr bool kNarrow = sizeof(CT) < 4;
  const uint32_t cnow = kNarrow ? nc.now : now;  // the value a touch writes
  __shared__ ScanTables t;
  load_scan_tables(t, tabs);
  const uint32_t now_slot = now % K;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(pairs) & 15u) == 0;
  const uint64_t pol_first = HINT ? l2_policy_first() : 0, pol_last = HINT ? l2_policy_last() : 0;
  constexpr uint32_t LB = BW == 8 ? 3 : BW == 4 ? 2 : 0;
  const uint32_t rb = 48u - (lg - LB), mask = (1u << (lg - LB)) - 1u;
  constexpr int P = SSPD_PIPE_PPT;
  constexpr uint32_t RM = R ? R : 8;
  const uint32_t nr = R ? R : geo.r;
  const uint64_t ngroups = (n + P - 1) / P;
  uint32_t n_fresh = 0;
  uint32_t pc[P], pb[P], p0[P];  // the previous group's fresh pairs: cip, bucket, row-0 column
  bool pv[P];
#pragma unroll
  for (int u = 0; u < P; ++u) pv[u] = false;
  // SSPD_CSET_PF: the next group's 16 B of pairs are loaded one iteration
  // ahead, so the stream's DRAM latency is off the probe chain
  constexpr bool kPf = SSPD_CSET_PF && P == 2;
  auto full_group = [&](uint64_t gg) { return gg < ngroups && vec && gg * P + P <= n; };
  uint4 nxt = make_uint4(0u, 0u, 0u, 0u);
  if (kPf && full_group(tid))
    nxt = HINT ? ld_stream_u4_hint(pairs + 2 * (tid * P), pol_first) : ld_stream_u4(pairs + 2 * (tid * P));
  // one extra round per thread drains the last group's pending stamps
  for (uint64_t g = tid; g < ngroups + nthreads; g += nthreads) {
    const bool have = g < ngroups;
    uint32_t c[P], o[P];
    bool valid[P];
    const uint64_t q0 = g * P;
    if (kPf && full_group(g)) {
      const uint4 a = nxt;
      const uint64_t gn = g + nthreads;
      if (full_group(gn))
        nxt = HINT ? ld_stream_u4_hint(pairs + 2 * (gn * P), pol_first) : ld_stream_u4(pairs + 2 * (gn * P));
      c[0] = a.x; o[0] = a.y; c[P - 1] = a.z; o[P - 1] = a.w;
      valid[0] = valid[P - 1] = true;
    } else if (P >= 2 && have && vec && q0 + P <= n) {
#pragma unroll
      for (int u = 0; u < P; u += 2) {
        const uint4 a = HINT ? ld_stream_u4_hint(pairs + 2 * (q0 + u), pol_first) : ld_stream_u4(pairs + 2 * (q0 + u));
        c[u] = a.x; o[u] = a.y; c[u + 1] = a.z; o[u + 1] = a.w;
        valid[u] = valid[u + 1] = true;
      }
    } else {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        valid[u] = have && q0 + u < n;
        c[u] = valid[u] ? pairs[2 * (q0 + u)] : 0u;
        o[u] = valid[u] ? pairs[2 * (q0 + u) + 1] : 0u;
      }
    }
    uint32_t b[P], home[P], rem[P], v[P];
    constexpr int BWL = BW == 1 ? 4 : BW;  // bucket type (unused when BW == 1)
    CBucket<BWL> vb[BW == 1 ? 1 : P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      b[u] = h1_bucket<H1MODE>(t, geo, o[u]);
      const uint64_t x = cset_perm48((uint64_t)c[u] << 16 | b[u]);
      home[u] = (uint32_t)(x >> rb);
      rem[u] = (uint32_t)x & ((1u << rb) - 1u);
      // PASSES: this launch takes only the keys whose home lies in its part
      // of the table (the top part_log2 bits of the home), so one pass's
      // probes touch 1/2^part_log2 of the set
      valid[u] = valid[u] && (home[u] >> part_shift) == part;
      if constexpr (BW == 1) {
        v[u] = valid[u] ? (HINT ? ld_ca_hint_u32(table + home[u], pol_last) : __ldca(table + home[u])) : 0u;
      } else {
        if (valid[u]) vb[u] = ld_bucket<BWL, HINT>(table + (uint64_t)home[u] * BW, pol_last);
      }
    }
    // the previous group's stamps, in flight together with this group's probes
    uint32_t old[P][RM];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (!pv[u]) continue;
#pragma unroll
      for (uint32_t row = 0; row < RM; ++row)
        if (row < nr) {
          const uint32_t cell = row << geo.q | row_col(geo, row, pc[u], p0[u]);
          CT* sp = stamps + (uint64_t)cell * geo.eta + pb[u];
          old[u][row] = cnow;
#if SSPD_AB_DIAG == 2
          // DIAGNOSTIC BUILD ONLY (wrong results): non-returning stamps, no ring
          if constexpr (!kNarrow)
            asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(sp), "r"(now) : "memory");
#else
          if (SSPD_OK_OR_SKIP(rec_ok(geo, cell, pb[u]))) {
            if constexpr (sizeof(CT) == 1) old[u][row] = narrow_max_from(sp, nc.now, word_of(sp));
            else if constexpr (kNarrow) old[u][row] = narrow_max(sp, nc.now);
            else old[u][row] = HINT ? atom_max_hint(sp, now, pol_first) : atomicMax(sp, now);
          }
#endif
        }
    }
    bool fresh[P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if constexpr (BW == 1)
        fresh[u] = valid[u] && cset_resolve(table, mask, home[u], rem[u], v[u]);
      else
        fresh[u] = valid[u] && cset_resolve_bucket<BWL, HINT>(table, mask, home[u], rem[u], rb, vb[u], pol_last);
    }
    // window ring moves for the previous group's first touches
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (!pv[u]) continue;
#pragma unroll
      for (uint32_t row = 0; row < RM; ++row) {
#if SSPD_AB_DIAG == 3
        n_fresh += (row < nr && old[u][row] == 0x7fffffffu);  // consume the returned stamps, no ring moves
        continue;
#endif
        if (SSPD_AB_DIAG || row >= nr || old[u][row] >= cnow) continue;  // diagnostic builds: no ring moves
        const uint32_t cell = row << geo.q | row_col(geo, row, pc[u], p0[u]);
        if constexpr (kNarrow) {
          narrow_ring(old[u][row], cell, nc, now, now_slot, geo, hist, K);
          continue;
        }
        ring_add(hist, now_slot, geo.ncells, cell, K, __LINE__);
        if (old[u][row] + K > now)
          ring_sub(hist, ring_back(now_slot, now - old[u][row], K), geo.ncells, cell, K, __LINE__);
      }
    }
    // this group's fresh pairs become pending
#pragma unroll
    for (int u = 0; u < P; ++u) {
      pv[u] = fresh[u];
      n_fresh += fresh[u];
      if (!fresh[u]) continue;
      pc[u] = c[u];
      pb[u] = b[u];
      p0[u] = row0_col(t, geo, c[u]);
    }
  }
  // keys new to this slot (set inserts plus probe-limit misses): one atomic per warp
  if (fresh_count) {
#pragma unroll
    for (int off = 16; off; off >>= 1) n_fresh += __shfl_xor_sync(0xffffffffu, n_fresh, off);
    if ((threadIdx.x & 31) == 0 && n_fresh) atomicAdd(fresh_count, (unsigned long long)n_fresh);
  }
}

// BINNING (partition pairs by pair-set region before a dedup scan).  Two
// passes over the input with identical chunking: a per-CTA histogram of
// regions, then a scatter into region-major order at offsets from an
// exclusive scan; the dedup kernel then walks the binned pairs in order.
__global__ void __launch_bounds__(256) bin_count_kernel(const uint32_t* __restrict__ pairs, uint64_t n,
                                                        uint64_t chunk, uint32_t* __restrict__ counts) {
  __shared__ uint32_t s_hist[kPairBins];
  for (int i = threadIdx.x; i < kPairBins; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(n, lo + chunk);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint2 p = *reinterpret_cast<const uint2*>(pairs + 2 * i);
    atomicAdd(&s_hist[pair_bin(pair_slot_hash((uint64_t)p.x << 32 | p.y))], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kPairBins; b += blockDim.x) counts[(uint64_t)b * gridDim.x + blockIdx.x] = s_hist[b];
}

// Exclusive scan of counts laid out [bin][cta] (one CTA, in place).
__global__ void __launch_bounds__(1024) bin_offsets_kernel(uint32_t* __restrict__ counts, uint32_t n_items) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t base = 0; base < n_items; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < n_items ? counts[i] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const uint32_t w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0u;
      uint32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      s_warp[lane] = wi - w;
    }
    __syncthreads();
    const uint32_t excl = s_carry + s_warp[wid] + incl - v;
    if (i < n_items) counts[i] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) bin_scatter_kernel(const uint32_t* __restrict__ pairs, uint64_t n,
                                                          uint64_t chunk, const uint32_t* __restrict__ offsets,
                                                          uint2* __restrict__ out) {
  __shared__ uint32_t s_pos[kPairBins];
  for (int b = threadIdx.x; b < kPairBins; b += blockDim.x)
    s_pos[b] = offsets[(uint64_t)b * gridDim.x + blockIdx.x];
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(n, lo + chunk);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint2 p = *reinterpret_cast<const uint2*>(pairs + 2 * i);
    const uint32_t pos = atomicAdd(&s_pos[pair_bin(pair_slot_hash((uint64_t)p.x << 32 | p.y))], 1u);
    out[pos] = p;
  }
}

// ---------------------------------------------------------------------------
// COMMIT: fold this slot's touched bitmap into the stamps (stamp = now) and,
// when a window of K slots is tracked, move each first-touched bucket's count
// from the ring entry of its previous stamp to the entry of `now`.  Clears
// the bitmap.  Each thread takes 4 bitmap words (128 recorders) per 16-byte
// load, skips empty groups, and walks its set bits; the stamp accesses of a
// warp stay within 16 KiB of address space, in order, so DRAM sees an ordered
// sparse stream rather than random scatter.
__device__ __forceinline__ void commit_word(uint32_t bits, uint64_t rec0, uint32_t* __restrict__ stamps,
                                            uint64_t n_rec, uint32_t now, uint32_t* __restrict__ hist,
                                            uint32_t K, uint32_t now_slot, uint32_t ncells, const Div40& by_eta) {
  while (bits) {
    const uint32_t b = __ffs(bits) - 1;
    bits &= bits - 1;
    const uint64_t rec = rec0 + b;
    if (rec >= n_rec) break;
    if (hist) {
      const uint32_t old = stamps[rec];
      if (old != now) {
        stamps[rec] = now;
        const uint32_t cell = (uint32_t)by_eta.div(rec);
        ring_add(hist, now_slot, ncells, cell, K, __LINE__);
        if (old + K > now) ring_sub(hist, ring_back(now_slot, now - old, K), ncells, cell, K, __LINE__);
      }
    } else {
      stamps[rec] = now;  // idempotent: a recorder touched this slot reads `now`
    }
  }
}

__global__ void __launch_bounds__(256) commit_kernel(uint32_t* __restrict__ touched, uint64_t nwords,
                                                     uint32_t* __restrict__ stamps, uint64_t n_rec,
                                                     uint32_t now, uint32_t* __restrict__ hist,
                                                     uint32_t K, uint32_t ncells, Div40 by_eta) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t now_slot = K ? now % K : 0;
  const uint64_t nvec = nwords >> 2;
  uint4* tv = reinterpret_cast<uint4*>(touched);
  for (uint64_t v = tid; v < nvec; v += nthreads) {
    const uint4 w = tv[v];
    if ((w.x | w.y | w.z | w.w) == 0) continue;
    tv[v] = make_uint4(0, 0, 0, 0);
    const uint64_t rec0 = v * 128;
    commit_word(w.x, rec0, stamps, n_rec, now, hist, K, now_slot, ncells, by_eta);
    commit_word(w.y, rec0 + 32, stamps, n_rec, now, hist, K, now_slot, ncells, by_eta);
    commit_word(w.z, rec0 + 64, stamps, n_rec, now, hist, K, now_slot, ncells, by_eta);
    commit_word(w.w, rec0 + 96, stamps, n_rec, now, hist, K, now_slot, ncells, by_eta);
  }
  for (uint64_t wi = nvec * 4 + tid; wi < nwords; wi += nthreads) {
    const uint32_t w = touched[wi];
    if (!w) continue;
    touched[wi] = 0;
    commit_word(w, wi * 32, stamps, n_rec, now, hist, K, now_slot, ncells, by_eta);
  }
}

// ---------------------------------------------------------------------------
// COUNT: rec::active_count per estimator (estimator.hpp:26-31) straight from
// the stamps: R_k(cell) = #{bucket : stamp > now - k}.  One warp per cell,
// 16-byte streaming loads when eta % 4 == 0.
__global__ void __launch_bounds__(256) count_kernel(const uint32_t* __restrict__ stamps, Geo geo,
                                                    uint32_t thr, uint32_t* __restrict__ counts) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec = (geo.eta & 3u) == 0;
  for (uint64_t cell = warp; cell < geo.ncells; cell += nwarps) {
    if (cell < geo.own_lo || cell >= geo.own_hi) {  // another router's cell: nothing here
      if (lane == 0) counts[cell] = 0;
      continue;
    }
    const uint32_t* est = stamps + cell * geo.eta;
    uint32_t c = 0;
    if (vec) {
      const uint32_t nq = geo.eta >> 2;
      uint32_t i = lane;
      for (; i + 32 < nq; i += 64) {
        const uint4 a = ld_stream_u4(est + 4 * i);
        const uint4 b = ld_stream_u4(est + 4 * (i + 32));
        c += (a.x > thr) + (a.y > thr) + (a.z > thr) + (a.w > thr);
        c += (b.x > thr) + (b.y > thr) + (b.z > thr) + (b.w > thr);
      }
      for (; i < nq; i += 32) {
        const uint4 a = ld_stream_u4(est + 4 * i);
        c += (a.x > thr) + (a.y > thr) + (a.z > thr) + (a.w > thr);
      }
    } else {
      for (uint32_t i = lane; i < geo.eta; i += 32) c += est[i] > thr;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[cell] = c;
  }
}

// R_k per cell from the tracked window ring: sum of the k most recent slots.
__global__ void hist_counts_kernel(const uint32_t* __restrict__ hist, uint32_t K, uint32_t ncells,
                                   uint32_t now, uint32_t k, uint32_t* __restrict__ counts) {
  for (uint32_t cell = blockIdx.x * blockDim.x + threadIdx.x; cell < ncells;
       cell += gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (uint32_t j = 0; j < k; ++j) c += hist[(uint64_t)((now - j) % K) * ncells + cell];
    counts[cell] = c;
  }
}

// Rebuild the window ring from the stamps (after imports or merges).
__global__ void __launch_bounds__(256) hist_rebuild_kernel(const uint32_t* __restrict__ stamps, Geo geo,
                                                           uint32_t now, uint32_t K,
                                                           uint32_t* __restrict__ hist) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t cell = warp; cell < geo.ncells; cell += nwarps) {
    if (cell < geo.own_lo || cell >= geo.own_hi) continue;
    const uint32_t* est = stamps + cell * geo.eta;
    for (uint32_t i = lane; i < geo.eta; i += 32) {
      const uint32_t s = est[i];
      if (s + K > now) atomicAdd(hist + (uint64_t)(s % K) * geo.ncells + cell, 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// HOT SETS, parallel form (two launches over all r*2^q cells).
// hot_mark: one thread per cell decides hot (R_k >= cutoff, with R_k from
// the per-cell counts or straight from the window ring) and publishes the
// hot bitmap word of its warp and the CTA's hot count.
// hot_write: each CTA adds up the counts of the row's earlier chunks and
// writes its hot columns in ascending order (rsea.cpp:65-84); the kernel
// also builds the transposed hot bits the joins index by key.
constexpr int kHotChunk = 1024;

// Programmatic dependent launch (the reconstruction chain is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): a kernel lets its
// successor start launching at once, and waits for its predecessor's results
// only where it first reads them.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(kHotChunk) hot_mark_kernel(const uint32_t* __restrict__ counts,
                                                            const uint32_t* __restrict__ hist, uint32_t K,
                                                            uint32_t now, uint32_t k, Geo geo, uint64_t cutoff,
                                                            uint32_t* __restrict__ hot_words,
                                                            uint32_t* __restrict__ chunk_counts, int from_words,
                                                            unsigned long long* __restrict__ zero,
                                                            uint32_t zero_words) {
  const uint32_t ncol = 1u << geo.q;
  // the reconstruction's bookkeeping starts at zero (one memset fewer)
  if (zero && blockIdx.x == 0)
    for (uint32_t i = threadIdx.x; i < zero_words; i += blockDim.x) zero[i] = 0ull;
  const uint32_t chunks = (ncol + kHotChunk - 1) / kHotChunk;
  const uint32_t row = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
  const uint32_t col = chunk * kHotChunk + threadIdx.x;
  const uint32_t cell = (row << geo.q) | col;
  const uint32_t wpr0 = (ncol + 31) / 32;
  bool hot = false;
  if (col < ncol && from_words) {
    // sharded routers: the hot bits were computed per owner and OR-merged
    hot = (hot_words[row * wpr0 + (col >> 5)] >> (col & 31)) & 1u;
  } else if (col < ncol) {
    uint32_t rk;
    if (hist) {
      rk = 0;
      for (uint32_t j = 0; j < k; ++j) rk += hist[(uint64_t)((now - j) % K) * geo.ncells + cell];
    } else {
      rk = counts[cell];
    }
    hot = rk >= cutoff;
  }
  const uint32_t b = __ballot_sync(0xffffffffu, hot);
  __shared__ uint32_t s_sum;
  if (threadIdx.x == 0) s_sum = 0;
  __syncthreads();
  const uint32_t wpr = (ncol + 31) / 32;  // words per row: rows never share a word
  if ((threadIdx.x & 31) == 0) {
    if (col < ncol && !from_words) hot_words[row * wpr + (col >> 5)] = b;
    if (b) atomicAdd(&s_sum, (uint32_t)__popc(b));
  }
  __syncthreads();
  if (threadIdx.x == 0) chunk_counts[blockIdx.x] = s_sum;
}

// Also writes the transposed hot bits the joins index by key:
// hotT[row][key][j / 32] bit j%32 = hot(row, col = j << (q - delta) | key).
__global__ void __launch_bounds__(kHotChunk) hot_write_kernel(const uint32_t* __restrict__ hot_words, Geo geo,
                                                             const uint32_t* __restrict__ chunk_counts,
                                                             uint32_t* __restrict__ cols_out,
                                                             uint32_t* __restrict__ row_counts,
                                                             uint32_t* __restrict__ hotT, uint32_t words_per_key) {
  pdl_trigger();
  pdl_wait();
  const uint32_t ncol = 1u << geo.q;
  const uint32_t chunks = (ncol + kHotChunk - 1) / kHotChunk;
  const uint32_t row = blockIdx.x / chunks, chunk = blockIdx.x % chunks;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __shared__ uint32_t s_base, s_warp[kHotChunk / 32];
  if (wid == 0) {
    uint32_t v = 0;
    for (uint32_t c = lane; c < chunk; c += 32) v += chunk_counts[row * chunks + c];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_base = v;
  }
  const uint32_t col = chunk * kHotChunk + threadIdx.x;
  const uint32_t wpr = (ncol + 31) / 32;
  const uint32_t w = col < ncol ? hot_words[row * wpr + (col >> 5)] : 0u;
  if (lane == 0) s_warp[wid] = __popc(w);
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = lane < kHotChunk / 32 ? s_warp[lane] : 0u;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    s_warp[lane] = incl - v;
  }
  __syncthreads();
  if ((w >> lane) & 1u)
    cols_out[(uint64_t)row * ncol + s_base + s_warp[wid] + __popc(w & ((1u << lane) - 1u))] = col;
  if (chunk == chunks - 1 && threadIdx.x == 0)
    row_counts[row] = s_base + chunk_counts[row * chunks + chunk];
  // transposed bits, one warp per word and one lane per bit (no atomics, so
  // no zeroing first)
  const uint32_t kbits = geo.q - geo.delta;
  const uint32_t seg_bits = 1u << geo.delta;
  const uint64_t per_row = (uint64_t)words_per_key << kbits;
  const uint64_t t_words = (uint64_t)geo.r * per_row;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < t_words; t += nwarps) {
    const uint32_t trow = (uint32_t)(t / per_row);
    const uint32_t rest = (uint32_t)(t % per_row);
    const uint32_t key = rest / words_per_key, j = (rest % words_per_key) * 32 + lane;
    const uint32_t c = (j << kbits) | key;
    const bool bit = j < seg_bits && ((hot_words[trow * wpr + (c >> 5)] >> (c & 31)) & 1u);
    const uint32_t b = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) hotT[t] = b;
  }
}

// ---------------------------------------------------------------------------
// RECONSTRUCTION joins (Alg. 6/7; rsea.cpp:179-237).  A tuple t of length m
// extends by row-m column c iff blocks_consistent(t0^t[m-1], t0^c), i.e.
// c & low_mask == ((t0 ^ t[m-1]) >> delta) ^ (t0 & low_mask): the matching
// columns are exactly the set bits of that key's row segment in hotT.  Every
// survivor is counted (64-bit, exact even past the cap, as CandidateOverflow
// reports it) and written while it fits the buffer.  Sizes come from device
// memory (row counts, previous level's count), so a whole reconstruction is
// queued without host round trips; a level whose input was truncated (count
// above the buffer) does nothing and the host re-runs with larger buffers.

// Device-side bookkeeping of one reconstruction, copied back in one piece.
struct ReconMeta {
  uint32_t rowcnt[64];             // hot columns per row
  unsigned long long level[64];    // survivors per level (index = level)
  unsigned long long surv;         // tuples passing the address checks
  unsigned long long pad[3];
};

__device__ __forceinline__ uint64_t warp_reserve(uint32_t mine, unsigned long long* counter,
                                                 uint32_t lane) {
  // inclusive warp scan of per-lane counts, one atomic per warp
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && total) base = atomicAdd(counter, (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - mine;
}

__device__ __forceinline__ uint32_t seg_popc(const uint32_t* seg, uint32_t words) {
  uint32_t c = 0;
  for (uint32_t w = 0; w < words; ++w) c += __popc(seg[w]);
  return c;
}

// Level 2: (c0, c1) over HSE(0) x HSE(1); c2 from row 2's segment.
__global__ void __launch_bounds__(256) level2_kernel(const uint32_t* __restrict__ cols, uint32_t ncol,
                                                     const uint32_t* __restrict__ T2, uint32_t wpk, Geo geo,
                                                     uint32_t* __restrict__ out, uint64_t out_cap,
                                                     ReconMeta* __restrict__ meta) {
  pdl_trigger();
  pdl_wait();
  const uint32_t n0 = meta->rowcnt[0], n1 = meta->rowcnt[1];
  const uint32_t* H0 = cols;
  const uint32_t* H1 = cols + ncol;
  unsigned long long* counter = &meta->level[2];
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t total = (uint64_t)n0 * n1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t kbits = geo.q - geo.delta;
  const uint32_t seg_bits = 1u << geo.delta;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < total; base += stride) {
    const uint64_t p = base + threadIdx.x;
    uint32_t c0 = 0, c1 = 0, key = 0, mine = 0;
    if (p < total) {
      c0 = H0[p / n1];
      c1 = H1[p % n1];
      key = (((c0 ^ c1) >> geo.delta) ^ (c0 & geo.low_mask));
      mine = seg_popc(T2 + (uint64_t)key * wpk, wpk);
    }
    uint64_t pos = warp_reserve(mine, counter, lane);
    if (mine) {
      const uint32_t* seg = T2 + (uint64_t)key * wpk;
      for (uint32_t w = 0; w < wpk; ++w) {
        uint32_t bits = seg[w];
        while (bits) {
          const uint32_t j = w * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          if (j >= seg_bits) break;
          if (pos < out_cap) {
            uint32_t* o = out + pos * 3;
            o[0] = c0;
            o[1] = c1;
            o[2] = key | (j << kbits);
          }
          ++pos;
        }
      }
    }
  }
}

// Levels 3..r-1: extend m-tuples by row m.
__global__ void __launch_bounds__(256) level_ext_kernel(const uint32_t* __restrict__ in, uint64_t in_cap,
                                                        uint32_t m, const uint32_t* __restrict__ Tm,
                                                        uint32_t wpk, Geo geo, uint32_t* __restrict__ out,
                                                        uint64_t out_cap, ReconMeta* __restrict__ meta) {
  pdl_trigger();
  pdl_wait();
  const uint64_t n_in = meta->level[m - 1];
  if (n_in > in_cap) return;  // input truncated: the host re-runs with larger buffers
  unsigned long long* counter = &meta->level[m];
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t kbits = geo.q - geo.delta;
  const uint32_t seg_bits = 1u << geo.delta;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n_in; base += stride) {
    const uint64_t t = base + threadIdx.x;
    uint32_t key = 0, mine = 0;
    const uint32_t* tup = in + t * m;
    if (t < n_in) {
      key = (((tup[0] ^ tup[m - 1]) >> geo.delta) ^ (tup[0] & geo.low_mask));
      mine = seg_popc(Tm + (uint64_t)key * wpk, wpk);
    }
    uint64_t pos = warp_reserve(mine, counter, lane);
    if (mine) {
      const uint32_t* seg = Tm + (uint64_t)key * wpk;
      for (uint32_t w = 0; w < wpk; ++w) {
        uint32_t bits = seg[w];
        while (bits) {
          const uint32_t j = w * 32 + __ffs(bits) - 1;
          bits &= bits - 1;
          if (j >= seg_bits) break;
          if (pos < out_cap) {
            uint32_t* o = out + pos * (m + 1);
            for (uint32_t x = 0; x < m; ++x) o[x] = tup[x];
            o[m] = key | (j << kbits);
          }
          ++pos;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// FINALIZE (rsea.cpp:86-108) in two kernels.  The accept set equals the
// reference's, which tests R_k first: the three tests are a conjunction.
//
// (1) address checks, one thread per r-tuple: assemble_ip (hashing.cpp:45-61)
//     then the row-0 re-hash; survivors are compacted.
__global__ void __launch_bounds__(256) finalize_check_kernel(const uint32_t* __restrict__ tuples,
                                                             uint64_t in_cap, const HashTabs* __restrict__ tabs,
                                                             Geo geo, ReconMeta* __restrict__ meta,
                                                             uint32_t* __restrict__ surv_idx,
                                                             uint32_t* __restrict__ surv_cip,
                                                             uint32_t* __restrict__ surv_rk) {
  pdl_trigger();
  __shared__ uint16_t s_row0[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    s_row0[i >> 8][i & 255] = (uint16_t)tabs->row0[i >> 8][i & 255];
  __syncthreads();
  pdl_wait();
  const uint64_t n = meta->level[geo.r - 1];
  if (n > in_cap) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint64_t t = base + threadIdx.x;
    bool ok = false;
    uint32_t ip = 0;
    if (t < n) {
      const uint32_t* cols = tuples + t * geo.r;
      const uint32_t c0 = cols[0];
      uint64_t acc = 0;
      for (uint32_t j = 0; j + 1 < geo.r; ++j) acc |= (uint64_t)(c0 ^ cols[j + 1]) << ((j * geo.delta) & 63u);
      ip = (uint32_t)acc;
      ok = true;
      for (uint32_t j = 0; j + 1 < geo.r; ++j)
        if ((shr32(ip, j * geo.delta) & geo.col_mask) != (c0 ^ cols[j + 1])) ok = false;
      if (ok) {
        const uint32_t h0 = ((uint32_t)s_row0[0][ip & 0xff] ^ s_row0[1][(ip >> 8) & 0xff] ^
                             s_row0[2][(ip >> 16) & 0xff] ^ s_row0[3][ip >> 24]) &
                            geo.col_mask;
        ok = (h0 == c0);
      }
    }
    const uint64_t pos = warp_reserve(ok ? 1u : 0u, &meta->surv, lane);
    if (ok) {
      surv_idx[pos] = (uint32_t)t;
      surv_cip[pos] = ip;
      if (surv_rk) surv_rk[pos] = 0;  // finalize_count adds into it
    }
  }
}

// (2) in-window count of the intersected estimator (max distance == min
//     stamp over the r rows), spread over CTAs: work item = (survivor, chunk
//     of 1024 buckets), 16-byte loads, one atomicAdd per CTA.
//     kmode: 0 -> stamp > thr, 1 -> nothing active (k == 0), 2 -> all (k > 65535).
__global__ void __launch_bounds__(256) finalize_count_kernel(const uint32_t* __restrict__ tuples,
                                                             const uint32_t* __restrict__ stamps, Geo geo,
                                                             uint32_t thr, int kmode,
                                                             const ReconMeta* __restrict__ meta,
                                                             const uint32_t* __restrict__ surv_idx,
                                                             uint32_t* __restrict__ surv_rk) {
  pdl_trigger();
  pdl_wait();
  constexpr uint32_t kChunk = 1024;
  const uint64_t n_surv = meta->surv;
  const uint32_t chunks = (geo.eta + kChunk - 1) / kChunk;
  __shared__ uint32_t s_cols[64];
  __shared__ uint32_t s_red[8];
  const bool vec = (geo.eta & 3u) == 0;
  for (uint64_t item = blockIdx.x; item < n_surv * chunks; item += gridDim.x) {
    const uint64_t sidx = item / chunks;
    const uint32_t c0 = (uint32_t)(item % chunks) * kChunk;
    const uint32_t c1 = min(c0 + kChunk, geo.eta);
    __syncthreads();
    if (threadIdx.x < geo.r) {
      s_cols[threadIdx.x] = tuples[(uint64_t)surv_idx[sidx] * geo.r + threadIdx.x];
      if (!SSPD_OK_OR_SKIP(s_cols[threadIdx.x] <= geo.col_mask)) s_cols[threadIdx.x] = 0;
    }
    __syncthreads();
    uint32_t cnt = 0;
    if (kmode == 0) {
      if (vec) {
        for (uint32_t b = c0 + 4 * threadIdx.x; b < c1; b += 4 * blockDim.x) {
          uint4 m = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
          for (uint32_t row = 0; row < geo.r; ++row) {
            const uint4 v = ld_stream_u4(stamps + ((uint64_t)row << geo.q | s_cols[row]) * geo.eta + b);
            m.x = min(m.x, v.x);
            m.y = min(m.y, v.y);
            m.z = min(m.z, v.z);
            m.w = min(m.w, v.w);
          }
          cnt += (m.x > thr) + (m.y > thr) + (m.z > thr) + (m.w > thr);
        }
      } else {
        for (uint32_t b = c0 + threadIdx.x; b < c1; b += blockDim.x) {
          uint32_t m = 0xffffffffu;
          for (uint32_t row = 0; row < geo.r; ++row)
            m = min(m, stamps[((uint64_t)row << geo.q | s_cols[row]) * geo.eta + b]);
          cnt += m > thr;
        }
      }
    } else if (kmode == 2) {
      for (uint32_t b = c0 + threadIdx.x; b < c1; b += blockDim.x) ++cnt;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += s_red[w];
      if (t) atomicAdd(surv_rk + sidx, t);
    }
  }
}

// ---------------------------------------------------------------------------
// EXACT GROUND TRUTH on the device: distinct opposite hosts
// per cip over one window of pairs -- what exact_counts computes with hash
// sets per slot and a trailing union (workload.cpp:180-213) -- by an exact
// set of (cip, oip) keys and a cip -> count map.  Probing is bounded by the
// table size; a full table raises `overflow` instead of looping.
__device__ __forceinline__ bool exact_pair_new(unsigned long long* __restrict__ pset, uint64_t pmask, uint64_t key,
                                               unsigned int* __restrict__ flags) {
  if (key == kEmptyKey) return atomicExch(&flags[1], 1u) == 0u;  // the one key equal to the marker
  const uint64_t h = pair_mix_hash(key);
  for (uint64_t i = 0; i <= pmask; ++i) {
    const uint64_t slot = (h + i) & pmask;
    const unsigned long long v = pset[slot];
    if (v == key) return false;
    if (v == kEmptyKey) {
      const unsigned long long old = atomicCAS(pset + slot, kEmptyKey, key);
      if (old == kEmptyKey) return true;
      if (old == key) return false;
    }
  }
  atomicExch(&flags[0], 1u);
  return false;
}

__global__ void __launch_bounds__(256) exact_insert_kernel(const uint32_t* __restrict__ pairs, uint64_t n,
                                                           unsigned long long* __restrict__ pset, uint64_t pmask,
                                                           unsigned long long* __restrict__ ckeys,
                                                           uint32_t* __restrict__ ccounts, uint64_t cmask,
                                                           unsigned int* __restrict__ flags) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t cip = pairs[2 * i], oip = pairs[2 * i + 1];
    if (!exact_pair_new(pset, pmask, (uint64_t)cip << 32 | oip, flags)) continue;
    const unsigned long long ck = (unsigned long long)cip + 1;  // 0 marks an empty slot
    uint64_t h = ck * 0x9e3779b97f4a7c15ull;
    h ^= h >> 31;
    bool placed = false;
    for (uint64_t j = 0; j <= cmask && !placed; ++j) {
      const uint64_t slot = (h + j) & cmask;
      unsigned long long v = ckeys[slot];
      if (v == 0ull) {
        const unsigned long long old = atomicCAS(ckeys + slot, 0ull, ck);
        v = old == 0ull ? ck : old;
      }
      if (v == ck) {
        atomicAdd(ccounts + slot, 1u);
        placed = true;
      }
    }
    if (!placed) atomicExch(&flags[0], 1u);
  }
}

__global__ void exact_emit_kernel(const unsigned long long* __restrict__ ckeys, const uint32_t* __restrict__ ccounts,
                                  uint64_t centries, uint32_t min_count, uint32_t* __restrict__ out_cip,
                                  uint32_t* __restrict__ out_count, uint64_t out_cap,
                                  unsigned long long* __restrict__ counter) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < centries;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ckeys[i];
    if (k == 0ull || ccounts[i] < min_count) continue;
    const unsigned long long pos = atomicAdd(counter, 1ull);
    if (pos < out_cap) {
      out_cip[pos] = (uint32_t)(k - 1);
      out_count[pos] = ccounts[i];
    }
  }
}

// ---------------------------------------------------------------------------
// Element-wise helpers.

// (ts, cip, oip) trace records (workload.hpp TraceRecord) -> (cip, oip) pairs.
__global__ void records_to_pairs_kernel(const uint32_t* __restrict__ rec, uint64_t n, uint2* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = make_uint2(rec[3 * i + 1], rec[3 * i + 2]);
}

__global__ void fill_u32_kernel(uint32_t* p, uint64_t n, uint32_t v) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// distance = min(now - stamp, 0xFFFF)
__global__ void stamps_to_dist_kernel(const uint32_t* __restrict__ s, uint64_t n, uint32_t now,
                                      uint16_t* __restrict__ d) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t age = now - s[i];
    d[i] = (uint16_t)(age < 0xffffu ? age : 0xffffu);
  }
}

// stamp = d == 0xFFFF ? 0 : now - d
__global__ void dist_to_stamps_kernel(const uint16_t* __restrict__ d, uint64_t n, uint32_t now,
                                      uint32_t* __restrict__ s) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = d[i];
    s[i] = v == 0xffffu ? 0u : now - v;
  }
}

// merge_rseas (snapshot.cpp:131-139) on stamps brought to a common `now`:
// union-min of distances == max of stamps, paper-max == min of stamps.
// `srcs` may point into peer devices' memory (NVLink loads).
struct MergeSrc {
  const uint32_t* p;
  uint32_t lag;  // common_now - this grid's now
};

__device__ __forceinline__ uint32_t rebase(uint32_t s, uint32_t now_common, uint32_t lag) {
  // distance in the source frame, saturated, re-expressed at now_common
  const uint32_t age = (now_common - lag) - s;
  const uint32_t d = age < 0xffffu ? age : 0xffffu;
  return d == 0xffffu ? 0u : now_common - d;
}

// Streams 16 bytes per source per step (every grid's stamps are 256-byte
// aligned); a scalar loop covers a tail of n % 4.
__global__ void __launch_bounds__(256) merge_kernel(const MergeSrc* __restrict__ srcs, uint32_t nsrc,
                                                    uint64_t n, uint32_t now_common, int take_max,
                                                    uint32_t* __restrict__ out) {
  auto pick = [&](uint32_t a, uint32_t v) { return take_max ? (v > a ? v : a) : (v < a ? v : a); };
  const uint64_t nv = n / 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
    const uint4 a0 = ld_stream_u4(srcs[0].p + 4 * i);
    const uint32_t l0 = srcs[0].lag;
    uint4 acc = make_uint4(rebase(a0.x, now_common, l0), rebase(a0.y, now_common, l0), rebase(a0.z, now_common, l0),
                           rebase(a0.w, now_common, l0));
    for (uint32_t g = 1; g < nsrc; ++g) {
      const uint4 v = ld_stream_u4(srcs[g].p + 4 * i);
      const uint32_t lg = srcs[g].lag;
      acc.x = pick(acc.x, rebase(v.x, now_common, lg));
      acc.y = pick(acc.y, rebase(v.y, now_common, lg));
      acc.z = pick(acc.z, rebase(v.z, now_common, lg));
      acc.w = pick(acc.w, rebase(v.w, now_common, lg));
    }
    reinterpret_cast<uint4*>(out)[i] = acc;
  }
  for (uint64_t i = nv * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint32_t acc = rebase(srcs[0].p[i], now_common, srcs[0].lag);
    for (uint32_t g = 1; g < nsrc; ++g) acc = pick(acc, rebase(srcs[g].p[i], now_common, srcs[g].lag));
    out[i] = acc;
  }
}

// Rsea::operator== on distances.
__global__ void equal_kernel(const uint32_t* __restrict__ a, uint32_t now_a, const uint32_t* __restrict__ b,
                             uint32_t now_b, uint64_t n, int* __restrict__ differ) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t da = now_a - a[i], db = now_b - b[i];
    da = da < 0xffffu ? da : 0xffffu;
    db = db < 0xffffu ? db : 0xffffu;
    if (da != db) {
      *differ = 1;
      return;
    }
  }
}

// ---------------------------------------------------------------------------
// SHARDED ROUTERS (union-min across N routers, each owning a contiguous 1/N
// slice of the cells; dist.py ShardExchange).  A router stamps only the
// recorders of cells it owns and pushes each pair new to it to the owners of
// its other cells (P2P stores into their inboxes), so per-router stamping
// scales with 1/N of the union of the routers' pairs instead of all of it.
// Hot sets are OR-merged across owners; a survivor's in-window count is the
// popcount of the AND, across owners, of per-owner bucket masks.
struct ShardArgs {
  uint2* const* inbox;            // device array of `world` inbox bases (peer-mapped)
  unsigned long long* sent;       // `world` counters: pairs pushed to each owner this slot
  uint32_t world, rank;
  uint64_t region_cap;            // pairs per (destination, source) region
};

// cell * world < 2^22 * 32: the 32-bit division is exact (and cheap next to
// a 64-bit one)
__device__ __forceinline__ uint32_t shard_owner(uint32_t cell, uint32_t ncells, uint32_t world) {
  return (cell * world) / ncells;
}

// PUSH = 1: the router's own pairs -- those it already saw this slot are
// skipped by the pair set, as in dedup mode; the rest stamp owned cells and
// are pushed to the other owners.  PUSH = 0: pairs received from peers go
// through the same pair set (a pair several routers saw arrives several
// times; at N=8 on C2 a router receives ~3 copies per distinct pair), then
// stamp owned cells only.
// Relayed routers (two hops, ShardExchange(relay=True)): own pairs go first
// to a pair owner (MODE 2: pair set, then one push per new pair, no
// stamping), which dedups the union of the routers' pairs for its share and
// relays each once to the cell owners (MODE 1 over the received lists, with
// a second pair set); cell owners stamp what arrives (MODE 4: no pair set --
// every pair reaches them once).
enum ShardMode { kShardRecv = 0, kShardOwn = 1, kShardToPairOwner = 2, kShardRecvOnce = 4 };

// Several inbox regions scanned as one input (one launch, so each warp pads
// its list blocks once, not once per region): logical pair i lies in segment
// s with start[s] <= i < start[s + 1], at pairs + 2 * (s * stride + i - start[s]).
struct ShardSegs {
  uint64_t stride;
  uint32_t nseg;  // 0: one contiguous input
  uint32_t skip;  // dev_counts: a segment read as empty (the router's own region), else ~0u
  uint64_t start[33];
  // Counts read by the kernel instead (no host round trip): segment i holds
  // dev_counts[i * count_stride] pairs -- e.g. a column of the all-gathered
  // per-router `sent` counters.  A count past `stride` is clamped and sets
  // *ovf (the caller checks it when it next synchronises).
  const unsigned long long* dev_counts;
  uint64_t count_stride;
  uint32_t* ovf;
};

__device__ __forceinline__ uint32_t pair_owner(uint64_t h, uint32_t world) {
  return (uint32_t)(h >> 32) % world;
}

template <int H1MODE, int HIST, int PUSH>
__global__ void __launch_bounds__(256) scan_shard_kernel(const uint32_t* __restrict__ pairs, uint64_t n,
                                                         const HashTabs* __restrict__ tabs, Geo geo,
                                                         unsigned long long* __restrict__ table, uint64_t table_mask,
                                                         uint32_t* __restrict__ stamps, uint32_t now,
                                                         uint32_t* __restrict__ hist, uint32_t K, ShardArgs sh,
                                                         ShardSegs segs = ShardSegs{}) {
  constexpr bool kPushes = PUSH == kShardOwn || PUSH == kShardToPairOwner;
  constexpr bool kStamps = PUSH != kShardToPairOwner;
  constexpr bool kDedup = PUSH != kShardRecvOnce;
  __shared__ ScanTables t;
  __shared__ ListState s_lists[8][kPushes ? 32 : 1];  // per warp (blockDim 256), per owner
  __shared__ uint64_t s_start[33];                     // segment starts (host or device counts)
  if (segs.nseg && threadIdx.x == 0) {
    uint64_t acc = 0;
    s_start[0] = 0;
    for (uint32_t i = 0; i < segs.nseg; ++i) {
      uint64_t c;
      if (segs.dev_counts) {
        c = i == segs.skip ? 0ull : segs.dev_counts[i * segs.count_stride];
        if (c > segs.stride) {
          if (segs.ovf) atomicOr(segs.ovf, 1u);
          c = segs.stride;
        }
      } else {
        c = segs.start[i + 1] - segs.start[i];
      }
      acc += c;
      s_start[i + 1] = acc;
    }
  }
  load_scan_tables(t, tabs);  // (its __syncthreads also publishes s_start)
  if (segs.nseg) n = s_start[segs.nseg];
  const uint32_t now_slot = HIST ? now % K : 0;
  const uint32_t lane = threadIdx.x & 31;
  ListState* wl = s_lists[threadIdx.x >> 5];
  if (kPushes)
    for (uint32_t d = 0; d < sh.world; ++d) list_init(wl[d], lane);
  constexpr int P = 2;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(pairs) & 15u) == 0;
  const uint64_t ngroups = (n + P - 1) / P;
  auto deliver = [&](uint32_t d, uint64_t pos, uint2 pr) {
    if (pos < sh.region_cap) sh.inbox[d][(uint64_t)sh.rank * sh.region_cap + pos] = pr;
  };
  for (uint64_t g = tid; g < ngroups; g += nthreads) {
    uint32_t c[P], o[P];
    bool fresh[P];
    const uint64_t p0 = g * P;
    if (segs.nseg) {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const uint64_t i = p0 + u;
        fresh[u] = i < n;
        c[u] = o[u] = 0u;
        if (fresh[u]) {
          uint32_t sg = 0;
          while (i >= s_start[sg + 1]) ++sg;
          const uint2 v = *reinterpret_cast<const uint2*>(pairs + 2 * (sg * segs.stride + (i - s_start[sg])));
          c[u] = v.x;
          o[u] = v.y;
        }
      }
    } else if (vec && p0 + P <= n) {
      const uint4 a = ld_stream_u4(pairs + 2 * p0);
      c[0] = a.x; o[0] = a.y; c[1] = a.z; o[1] = a.w;
      fresh[0] = fresh[1] = true;
    } else {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        fresh[u] = p0 + u < n;
        c[u] = fresh[u] ? pairs[2 * (p0 + u)] : 0u;
        o[u] = fresh[u] ? pairs[2 * (p0 + u) + 1] : 0u;
      }
    }
    uint32_t dmask[P] = {0u, 0u};
    if (kDedup) {
      uint64_t key[P], h[P];
      unsigned long long v[P];
#pragma unroll
      for (int u = 0; u < P; ++u) {
        key[u] = (uint64_t)c[u] << 32 | o[u];
        h[u] = pair_slot_hash(key[u]);
        v[u] = fresh[u] ? __ldca(table + pair_slot(h[u], 0, table_mask)) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < P; ++u) {
        fresh[u] = fresh[u] && pair_resolve(table, table_mask, key[u], h[u], v[u]);
        if (PUSH == kShardToPairOwner && fresh[u]) dmask[u] = 1u << pair_owner(h[u], sh.world);
      }
    }
#pragma unroll
    for (int u = 0; u < P; ++u) {
      if (!kStamps || !fresh[u]) continue;
      uint32_t bucket, col0;
      hash_pair<H1MODE>(t, geo, c[u], o[u], bucket, col0);
      for (uint32_t r0 = 0; r0 < geo.r; r0 += 8) {
        uint32_t cell[8], old[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {  // owned touches: atomics issued together
          const uint32_t row = r0 + j;
          old[j] = now;
          cell[j] = row << geo.q | row_col(geo, row, c[u], col0);
          if (row >= geo.r) continue;
          const uint32_t owner = shard_owner(cell[j], geo.ncells, sh.world);
          if (owner != sh.rank) {
            dmask[u] |= 1u << owner;
            continue;
          }
          if (!SSPD_OK_OR_SKIP(rec_ok(geo, cell[j], bucket))) continue;
          uint32_t* p = stamps + (uint64_t)cell[j] * geo.eta + bucket;
          if (HIST) old[j] = atomicMax(p, now);
          else asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(now) : "memory");
        }
        if (HIST) {
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j) {
            if (old[j] >= now) continue;
            ring_add(hist, now_slot, geo.ncells, cell[j], K, __LINE__);
            if (old[j] + K > now) ring_sub(hist, ring_back(now_slot, now - old[j], K), geo.ncells, cell[j], K, __LINE__);
          }
        }
      }
    }
    if (kPushes) {
      // block-reserved list per owner (list_append)
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const unsigned m = __activemask();
        // only the owners some lane of the warp sends to
        for (unsigned todo = __reduce_or_sync(m, dmask[u]); todo; todo &= todo - 1) {
          const uint32_t d = __ffs(todo) - 1;
          const bool mine = (dmask[u] >> d) & 1u;
          const uint2 pr = make_uint2(c[u], o[u]);
          const uint64_t pos = list_append(wl[d], sh.sent + d, m, mine, pr, lane);
          if (mine) deliver(d, pos, pr);
        }
      }
    }
  }
  if (kPushes) {
    for (uint32_t d = 0; d < sh.world; ++d) list_pad(wl[d], lane, [&](uint64_t pos, uint2 pr) { deliver(d, pos, pr); });
    __threadfence_system();  // peer stores visible before the exchange's barrier
  }
}

// Per survivor and 32-bucket word: the AND over the survivor's owned rows of
// "in window" (stamp > thr); rows owned elsewhere contribute all ones, so the
// AND across routers of these masks is the intersected estimator's bitmap.
// kmode as finalize_count_kernel.  Bits past eta are 0.
__global__ void __launch_bounds__(256) shard_mask_kernel(const uint32_t* __restrict__ tuples,
                                                         const uint32_t* __restrict__ stamps, Geo geo, uint32_t thr,
                                                         int kmode, const ReconMeta* __restrict__ meta,
                                                         const uint32_t* __restrict__ surv_idx, uint32_t world,
                                                         uint32_t rank, uint32_t* __restrict__ masks) {
  const uint32_t W = (geo.eta + 31) / 32;
  const uint64_t n = meta->surv * W;
  for (uint64_t item = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; item < n;
       item += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t sidx = item / W;
    const uint32_t w = (uint32_t)(item % W);
    const uint32_t nb = min(32u, geo.eta - w * 32);
    const uint32_t valid = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
    uint32_t m = kmode == 1 ? 0u : valid;
    if (kmode == 0) {
      const uint32_t* cols = tuples + (uint64_t)surv_idx[sidx] * geo.r;
      for (uint32_t row = 0; row < geo.r && m; ++row) {
        const uint32_t cell = row << geo.q | cols[row];
        if (shard_owner(cell, geo.ncells, world) != rank) continue;
        if (!SSPD_OK_OR_SKIP(rec_ok(geo, cell, w * 32 + nb - 1))) continue;
        const uint32_t* e = stamps + (uint64_t)cell * geo.eta + w * 32;
        uint32_t bits = 0;
        for (uint32_t j = 0; j < nb; ++j) bits |= (uint32_t)(e[j] > thr) << j;
        m &= bits;
      }
    }
    masks[item] = m;
  }
}

// dst = OR / AND over up to 32 source word arrays (peer memory allowed), 16 B
// at a time where every pointer is aligned.
struct ReduceSrcs {
  const uint32_t* p[32];
};
template <int AND>
__global__ void __launch_bounds__(256) reduce_words_kernel(ReduceSrcs srcs, uint32_t n_src, uint64_t words,
                                                           uint32_t* __restrict__ dst, int vec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (vec) {
    for (uint64_t i = tid; i < words / 4; i += stride) {
      uint4 acc = AND ? make_uint4(~0u, ~0u, ~0u, ~0u) : make_uint4(0u, 0u, 0u, 0u);
      for (uint32_t s = 0; s < n_src; ++s) {
        const uint4 v = __ldcv(reinterpret_cast<const uint4*>(srcs.p[s]) + i);  // peers' fresh data
        if (AND) acc.x &= v.x, acc.y &= v.y, acc.z &= v.z, acc.w &= v.w;
        else acc.x |= v.x, acc.y |= v.y, acc.z |= v.z, acc.w |= v.w;
      }
      reinterpret_cast<uint4*>(dst)[i] = acc;
    }
    for (uint64_t i = words / 4 * 4 + tid; i < words; i += stride) {
      uint32_t acc = AND ? ~0u : 0u;
      for (uint32_t s = 0; s < n_src; ++s) acc = AND ? (acc & __ldcv(srcs.p[s] + i)) : (acc | __ldcv(srcs.p[s] + i));
      dst[i] = acc;
    }
    return;
  }
  for (uint64_t i = tid; i < words; i += stride) {
    uint32_t acc = AND ? ~0u : 0u;
    for (uint32_t s = 0; s < n_src; ++s) acc = AND ? (acc & __ldcv(srcs.p[s] + i)) : (acc | __ldcv(srcs.p[s] + i));
    dst[i] = acc;
  }
}

// R_k of each survivor = popcount of its merged mask (one warp per survivor).
__global__ void shard_popcount_kernel(const uint32_t* __restrict__ masks, const ReconMeta* __restrict__ meta,
                                      uint32_t W, uint32_t* __restrict__ surv_rk) {
  const uint64_t n = meta->surv;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < n;
       s += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    uint32_t c = 0;
    for (uint32_t w = lane; w < W; w += 32) c += __popc(masks[s * W + w]);
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) surv_rk[s] = c;
  }
}

// ---------------------------------------------------------------------------
// NARROW STAMPS (w = 8 or 16 bits per recorder; BASELINE config C4's
// stamp-width axis).  Exactness domain: in-window counts R_k for k <= K (the
// grid's window, fixed at creation) and everything derived from them (hot
// sets, finalize, reconstruction reports); full distances are not kept.
//
// Codes rise with time inside an epoch: 0 = not seen in the window, and slot
// `s` writes code(s) = lo + (s - epoch0), so a recorder's age is
// code(now) - c.  Before code(now) would pass `hi`, a rebase pass
// (narrow_rebase_kernel) clears codes older than K and shifts the rest so
// that code(now) = lo + K - 1: an epoch lasts hi - lo - K + 2 slots.
//   w = 16: lo = 0x0080, hi = 0x7F7F -- the positive normal bf16 bit
//           patterns, which order like the integers, so a touch is ONE
//           returning packed-bf16 max atomic (ATOMG.E.MAX.BF16x2) whose other
//           lane is +0.0 (a no-op), like the 32-bit atomicMax; by default an
//           ld.cg of the code goes first (PRELOAD), so the atomic hits L2.
//   w = 8:  lo = 1, hi = 255; no 8-bit atomic exists, so a touch is a load
//           of the 32-bit word and a CAS on it (retried if a neighbour moved).
// The old code drives the window ring exactly as in the 32-bit scan.

// Scan into a narrow grid: direct stamping, optionally behind the per-slot
// pair set (DEDUP) of scan_dedup_kernel; 2 pairs per thread, every touch's
// atomic issued before any old code is consumed.  The window ring is always
// kept.  (A narrow grid's dedup scan normally runs scan_cset_kernel on its
// codes instead -- profiles/r02_ab_keyset.md A/Bs 16-17; this kernel is the
// direct scan and the $SSPD_CSET=0 / $SSPD_CSET8=0 dedup path.)
template <class T, int H1MODE, int DEDUP, int PRELOAD = 0>
__global__ void __launch_bounds__(256) scan_narrow_kernel(const uint32_t* __restrict__ pairs, uint64_t n,
                                                          const HashTabs* __restrict__ tabs, Geo geo,
                                                          unsigned long long* __restrict__ table, uint64_t table_mask,
                                                          T* __restrict__ codes, uint32_t now, NarrowCodes nc,
                                                          uint32_t* __restrict__ hist, uint32_t K) {
  __shared__ ScanTables t;
  load_scan_tables(t, tabs);
  const uint32_t now_slot = now % K;
  constexpr int P = 2;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(pairs) & 15u) == 0;
  const uint64_t ngroups = (n + P - 1) / P;
  for (uint64_t g = tid; g < ngroups; g += nthreads) {
    uint32_t c[P], o[P];
    bool fresh[P];
    const uint64_t p0 = g * P;
    if (vec && p0 + P <= n) {
      const uint4 a = ld_stream_u4(pairs + 2 * p0);
      c[0] = a.x; o[0] = a.y; c[1] = a.z; o[1] = a.w;
      fresh[0] = fresh[1] = true;
    } else {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        fresh[u] = p0 + u < n;
        c[u] = fresh[u] ? pairs[2 * (p0 + u)] : 0u;
        o[u] = fresh[u] ? pairs[2 * (p0 + u) + 1] : 0u;
      }
    }
    if (DEDUP) {
      uint64_t key[P], h[P];
      unsigned long long v[P];
#pragma unroll
      for (int u = 0; u < P; ++u) {
        key[u] = (uint64_t)c[u] << 32 | o[u];
        h[u] = pair_slot_hash(key[u]);
        v[u] = fresh[u] ? __ldca(table + pair_slot(h[u], 0, table_mask)) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < P; ++u) fresh[u] = fresh[u] && pair_resolve(table, table_mask, key[u], h[u], v[u]);
    }
    if (geo.r <= 8) {
      uint32_t bucket[P], col0[P], old[P][8];
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (!fresh[u]) continue;
        hash_pair<H1MODE>(t, geo, c[u], o[u], bucket[u], col0[u]);
#pragma unroll
        for (uint32_t row = 0; row < 8; ++row) {
          if (row >= geo.r) break;
          (void)SSPD_OK_OR_SKIP(rec_ok(geo, row << geo.q | row_col(geo, row, c[u], col0[u]), bucket[u]));
          T* p = codes + (uint64_t)(row << geo.q | row_col(geo, row, c[u], col0[u])) * geo.eta + bucket[u];
          if constexpr (sizeof(T) == 2 && !PRELOAD) old[u][row] = narrow_max(p, nc.now);
          else if constexpr (sizeof(T) == 2) old[u][row] = __ldcg(reinterpret_cast<const unsigned short*>(p));
          else old[u][row] = word_of(p);
        }
      }
      if constexpr (sizeof(T) == 2 && PRELOAD) {
        // the load pulled the line into L2: the atomic now hits there
#pragma unroll
        for (int u = 0; u < P; ++u) {
          if (!fresh[u]) continue;
#pragma unroll
          for (uint32_t row = 0; row < 8; ++row) {
            if (row >= geo.r) break;
            if (old[u][row] >= nc.now) continue;
            T* p = codes + (uint64_t)(row << geo.q | row_col(geo, row, c[u], col0[u])) * geo.eta + bucket[u];
            old[u][row] = narrow_max(p, nc.now);
          }
        }
      }
      if constexpr (sizeof(T) == 1) {
#pragma unroll
        for (int u = 0; u < P; ++u) {
          if (!fresh[u]) continue;
#pragma unroll
          for (uint32_t row = 0; row < 8; ++row) {
            if (row >= geo.r) break;
            T* p = codes + (uint64_t)(row << geo.q | row_col(geo, row, c[u], col0[u])) * geo.eta + bucket[u];
            old[u][row] = narrow_max_from(p, nc.now, old[u][row]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (!fresh[u]) continue;
#pragma unroll
        for (uint32_t row = 0; row < 8; ++row) {
          if (row >= geo.r) break;
          narrow_ring(old[u][row], row << geo.q | row_col(geo, row, c[u], col0[u]), nc, now, now_slot, geo, hist,
                      K);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (!fresh[u]) continue;
        uint32_t bucket, col0;
        hash_pair<H1MODE>(t, geo, c[u], o[u], bucket, col0);
        for (uint32_t row = 0; row < geo.r; ++row) {
          const uint32_t cell = row << geo.q | row_col(geo, row, c[u], col0);
          (void)SSPD_OK_OR_SKIP(rec_ok(geo, cell, bucket));
          T* p = codes + (uint64_t)cell * geo.eta + bucket;
          uint32_t old;
          if constexpr (sizeof(T) == 2) old = narrow_max(p, nc.now);
          else old = narrow_max_from(p, nc.now, word_of(p));
          narrow_ring(old, cell, nc, now, now_slot, geo, hist, K);
        }
      }
    }
  }
}

// Epoch rebase: codes older than K become 0, the rest move down by `shift`
// (streaming pass, 16-byte words).
template <class T>
__global__ void __launch_bounds__(256) narrow_rebase_kernel(T* __restrict__ codes, uint64_t n, uint32_t code_now,
                                                            uint32_t lo, uint32_t K, uint32_t shift) {
  constexpr uint32_t per = 16 / sizeof(T);
  const uint64_t nvec = n / per;
  uint4* v = reinterpret_cast<uint4*>(codes);
  auto fix = [&](uint32_t c) -> uint32_t {
    if (c < lo || code_now - c >= K) return 0u;
    return c - shift;
  };
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 x = v[i];
    T* e = reinterpret_cast<T*>(&x);
    bool dirty = false;
#pragma unroll
    for (uint32_t j = 0; j < per; ++j) {
      const uint32_t f = fix(e[j]);
      dirty |= f != e[j];
      e[j] = (T)f;
    }
    if (dirty) v[i] = x;
  }
  for (uint64_t i = nvec * per + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    codes[i] = (T)fix(codes[i]);
}

// finalize_count_kernel over narrow codes: a bucket counts when all r rows
// hold a live code younger than k (max distance < k), i.e. min code > thr
// with thr = code(now) - k clamped below lo.
template <class T>
__global__ void __launch_bounds__(256) finalize_count_narrow_kernel(const uint32_t* __restrict__ tuples,
                                                                    const T* __restrict__ codes, Geo geo,
                                                                    uint32_t thr, int kmode,
                                                                    const ReconMeta* __restrict__ meta,
                                                                    const uint32_t* __restrict__ surv_idx,
                                                                    uint32_t* __restrict__ surv_rk) {
  pdl_trigger();
  pdl_wait();
  constexpr uint32_t kChunk = 1024;
  const uint64_t n_surv = meta->surv;
  const uint32_t chunks = (geo.eta + kChunk - 1) / kChunk;
  __shared__ uint32_t s_cols[64];
  __shared__ uint32_t s_red[8];
  for (uint64_t item = blockIdx.x; item < n_surv * chunks; item += gridDim.x) {
    const uint64_t sidx = item / chunks;
    const uint32_t c0 = (uint32_t)(item % chunks) * kChunk;
    const uint32_t c1 = min(c0 + kChunk, geo.eta);
    __syncthreads();
    if (threadIdx.x < geo.r) s_cols[threadIdx.x] = tuples[(uint64_t)surv_idx[sidx] * geo.r + threadIdx.x];
    __syncthreads();
    uint32_t cnt = 0;
    if (kmode == 0) {
      for (uint32_t b = c0 + threadIdx.x; b < c1; b += blockDim.x) {
        uint32_t m = 0xffffffffu;
        for (uint32_t row = 0; row < geo.r; ++row)
          m = min(m, (uint32_t)codes[((uint64_t)row << geo.q | s_cols[row]) * geo.eta + b]);
        cnt += m > thr;
      }
    } else if (kmode == 2) {
      for (uint32_t b = c0 + threadIdx.x; b < c1; b += blockDim.x) ++cnt;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tt = 0;
      for (uint32_t w = 0; w < blockDim.x / 32; ++w) tt += s_red[w];
      if (tt) atomicAdd(surv_rk + sidx, tt);
    }
  }
}

}  // namespace sspd_dev
