// kernels.cuh -- sm_100a kernels for the sliding super point detector.
//
// Data layout in HBM:
//   stamps  u32[r * 2^q * eta]   (row, column, bucket) order, like the
//                                 reference's cells_ (rsea.hpp:105-112)
//   touched u32[ceil(n/32)]      this slot's touched recorders, 1 bit each
//   hist    u32[K * r * 2^q]     per-cell count of buckets whose latest touch
//                                 is slot s, ring-indexed by s mod K (optional)
// A recorder's reference distance is min(now - stamp, 0xFFFF); stamp 0 is
// never-seen and `now` starts at 65535.
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
  uint32_t eta_shift;    // log2(eta) when eta is a power of two, else 0xFF
  uint32_t ncells;       // r * 2^q
  uint64_t n_rec;        // ncells * eta
};

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

__device__ __forceinline__ uint2 ld_stream_u2(const void* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p));
  return v;
}

// ---------------------------------------------------------------------------
// SCAN: Rsea::update over a batch (rsea.cpp:29-53), recording touches in the
// per-slot bitmap.  The bitmap is 1/32 of the stamp grid; when it fits in L2
// (reference geometry: 20 MiB) every touch is an L2-resident red.or.
//
// H1MODE 0: eta a power of two <= 2^32, H1 needs only its low 32 bits.
// H1MODE 1: general eta, full 64-bit tabulation value % eta (hashing.hpp:58).
template <int H1MODE>
__global__ void __launch_bounds__(256) scan_bitmap_kernel(const uint32_t* __restrict__ pairs,
                                                          uint64_t n, const HashTabs* __restrict__ tabs,
                                                          Geo geo, uint32_t* __restrict__ touched) {
  __shared__ uint16_t s_row0[4][256];
  __shared__ uint64_t s_h1[4][256];  // low 32 bits used in mode 0
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    s_row0[i >> 8][i & 255] = (uint16_t)tabs->row0[i >> 8][i & 255];
    s_h1[i >> 8][i & 255] = tabs->h1[i >> 8][i & 255];
  }
  __syncthreads();
  const uint32_t* s_h1_lo = reinterpret_cast<const uint32_t*>(&s_h1[0][0]);

  auto touch = [&](uint32_t cip, uint32_t oip) {
    uint32_t bucket;
    if (H1MODE == 0) {
      // low words of the u64 entries (little endian): index 2*i
      uint32_t h = s_h1_lo[2 * (0 * 256 + (oip & 0xff))] ^ s_h1_lo[2 * (1 * 256 + ((oip >> 8) & 0xff))] ^
                   s_h1_lo[2 * (2 * 256 + ((oip >> 16) & 0xff))] ^ s_h1_lo[2 * (3 * 256 + (oip >> 24))];
      bucket = h & (geo.eta - 1u);
    } else {
      uint64_t h = s_h1[0][oip & 0xff] ^ s_h1[1][(oip >> 8) & 0xff] ^ s_h1[2][(oip >> 16) & 0xff] ^
                   s_h1[3][oip >> 24];
      bucket = (uint32_t)(h % geo.eta);
    }
    const uint32_t col0 = ((uint32_t)s_row0[0][cip & 0xff] ^ s_row0[1][(cip >> 8) & 0xff] ^
                           s_row0[2][(cip >> 16) & 0xff] ^ s_row0[3][cip >> 24]) &
                          geo.col_mask;
    // row 0
    uint64_t idx = (uint64_t)col0 * geo.eta + bucket;
    red_or(touched + (idx >> 5), 1u << (idx & 31));
    for (uint32_t row = 1; row < geo.r; ++row) {
      const uint32_t col = (shr32(cip, (row - 1) * geo.delta) ^ col0) & geo.col_mask;
      idx = ((uint64_t)row << geo.q | col) * geo.eta + bucket;
      red_or(touched + (idx >> 5), 1u << (idx & 31));
    }
  };

  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const bool aligned16 = ((reinterpret_cast<uintptr_t>(pairs) & 15u) == 0);
  if (aligned16) {
    // Two pairs per 16-byte load; two loads in flight per thread.
    const uint64_t nquads = n >> 1;
    uint64_t i = tid;
    for (; i + nthreads < nquads; i += 2 * nthreads) {
      const uint4 a = ld_stream_u4(pairs + 4 * i);
      const uint4 b = ld_stream_u4(pairs + 4 * (i + nthreads));
      touch(a.x, a.y);
      touch(a.z, a.w);
      touch(b.x, b.y);
      touch(b.z, b.w);
    }
    for (; i < nquads; i += nthreads) {
      const uint4 a = ld_stream_u4(pairs + 4 * i);
      touch(a.x, a.y);
      touch(a.z, a.w);
    }
    if ((n & 1) && tid == 0) touch(pairs[2 * (n - 1)], pairs[2 * (n - 1) + 1]);
  } else {
    for (uint64_t i = tid; i < n; i += nthreads) touch(pairs[2 * i], pairs[2 * i + 1]);
  }
}

// ---------------------------------------------------------------------------
// COMMIT: fold this slot's touched bitmap into the stamps (stamp = now) and,
// when a window of K slots is tracked, move each first-touched bucket's count
// from the ring entry of its previous stamp to the entry of `now`.  Clears
// the bitmap.  One warp covers 32 consecutive bitmap words (1024 recorders);
// for each non-zero word the lanes update the 32 recorders of that word, so
// the stamp writes of a warp land in one 128-byte line, in address order.
__global__ void __launch_bounds__(256) commit_kernel(uint32_t* __restrict__ touched, uint64_t nwords,
                                                     uint32_t* __restrict__ stamps, uint64_t n_rec,
                                                     uint32_t now, uint32_t* __restrict__ hist,
                                                     uint32_t K, uint32_t ncells, Div40 by_eta) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t now_slot = K ? now % K : 0;
  for (uint64_t base = warp * 32; base < nwords; base += nwarps * 32) {
    const uint64_t my = base + lane;
    uint32_t w = my < nwords ? touched[my] : 0u;
    uint32_t nz = __ballot_sync(0xffffffffu, w != 0);
    if (w) touched[my] = 0u;
    while (nz) {
      const int src = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint32_t word = __shfl_sync(0xffffffffu, w, src);
      const uint64_t rec = (base + src) * 32 + lane;
      if ((word >> lane) & 1u) {
        if (rec < n_rec) {
          const uint32_t old = stamps[rec];
          if (old != now) {
            stamps[rec] = now;
            if (hist) {
              const uint32_t cell = (uint32_t)by_eta.div(rec);
              atomicAdd(hist + (uint64_t)now_slot * ncells + cell, 1u);
              if (old + K > now) atomicSub(hist + (uint64_t)(old % K) * ncells + cell, 1u);
            }
          }
        }
      }
    }
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
    const uint32_t* est = stamps + cell * geo.eta;
    for (uint32_t i = lane; i < geo.eta; i += 32) {
      const uint32_t s = est[i];
      if (s + K > now) atomicAdd(hist + (uint64_t)(s % K) * geo.ncells + cell, 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// HOT SETS: ordered compaction of hot columns per row (rsea.cpp:65-84) and a
// transposed hot bitmap for the reconstruction joins: for key = col & low_mask
// and j = col >> (q - delta), bit j of the 2^delta-bit row segment of key.
// One CTA per row, 1024 threads.
__global__ void __launch_bounds__(1024) hot_compact_kernel(const uint32_t* __restrict__ counts, Geo geo,
                                                           uint64_t cutoff, uint32_t* __restrict__ cols_out,
                                                           uint32_t* __restrict__ row_counts,
                                                           uint32_t* __restrict__ hotT,
                                                           uint32_t words_per_key) {
  const uint32_t row = blockIdx.x;
  const uint32_t ncol = 1u << geo.q;
  const uint32_t kbits = geo.q - geo.delta;
  uint32_t* myT = hotT + (uint64_t)row * ((uint64_t)words_per_key << kbits);
  uint32_t* myCols = cols_out + (uint64_t)row * ncol;
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t c0 = 0; c0 < ncol; c0 += blockDim.x) {
    const uint32_t col = c0 + threadIdx.x;
    const bool hot = col < ncol && counts[(uint64_t)row * ncol + col] >= cutoff;
    const uint32_t b = __ballot_sync(0xffffffffu, hot);
    if (lane == 0) s_warp[wid] = __popc(b);
    __syncthreads();
    if (wid == 0) {
      uint32_t v = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      s_warp[lane] = incl - v;  // exclusive
    }
    __syncthreads();
    const uint32_t pos = s_base + s_warp[wid] + __popc(b & ((1u << lane) - 1u));
    if (hot) {
      myCols[pos] = col;
      const uint32_t key = col & geo.low_mask;
      const uint32_t j = col >> kbits;
      atomicOr(myT + (uint64_t)key * words_per_key + (j >> 5), 1u << (j & 31));
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_base = pos + (hot ? 1u : 0u);
    __syncthreads();
  }
  if (threadIdx.x == 0) row_counts[row] = s_base;
}

// ---------------------------------------------------------------------------
// RECONSTRUCTION joins (Alg. 6/7; rsea.cpp:179-237).  A tuple t of length m
// extends by row-m column c iff blocks_consistent(t0^t[m-1], t0^c), i.e.
// c & low_mask == ((t0 ^ t[m-1]) >> delta) ^ (t0 & low_mask): the matching
// columns are exactly the set bits of that key's row segment in hotT.  Every
// survivor is counted (64-bit, exact even past the cap, as CandidateOverflow
// reports it) and written while it fits the buffer.

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
__global__ void __launch_bounds__(256) level2_kernel(const uint32_t* __restrict__ H0, uint32_t n0,
                                                     const uint32_t* __restrict__ H1, uint32_t n1,
                                                     const uint32_t* __restrict__ T2, uint32_t wpk,
                                                     Geo geo, uint32_t* __restrict__ out,
                                                     uint64_t out_cap,
                                                     unsigned long long* __restrict__ counter) {
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
__global__ void __launch_bounds__(256) level_ext_kernel(const uint32_t* __restrict__ in, uint64_t n_in,
                                                        uint32_t m, const uint32_t* __restrict__ Tm,
                                                        uint32_t wpk, Geo geo, uint32_t* __restrict__ out,
                                                        uint64_t out_cap,
                                                        unsigned long long* __restrict__ counter) {
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
// FINALIZE (rsea.cpp:86-108), one warp per r-tuple.  The address checks
// (assemble_ip, hashing.cpp:45-61, then the row-0 re-hash) need no memory and
// run first; surviving tuples intersect their r estimators (max distance ==
// min stamp) and count in-window buckets.  The accept set equals the
// reference's, which tests R_k first: the three tests are a conjunction.
__global__ void __launch_bounds__(256) finalize_kernel(const uint32_t* __restrict__ tuples, uint64_t n,
                                                       const uint32_t* __restrict__ stamps,
                                                       const HashTabs* __restrict__ tabs, Geo geo,
                                                       uint32_t thr, uint64_t cutoff,
                                                       uint32_t* __restrict__ out_idx,
                                                       uint32_t* __restrict__ out_cip,
                                                       uint32_t* __restrict__ out_rk,
                                                       unsigned long long* __restrict__ counter,
                                                       uint8_t* __restrict__ accepted) {
  __shared__ uint16_t s_row0[4][256];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x)
    s_row0[i >> 8][i & 255] = (uint16_t)tabs->row0[i >> 8][i & 255];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = warp; t < n; t += nwarps) {
    const uint32_t* cols = tuples + t * geo.r;
    // assemble_ip over blocks B(i) = c0 ^ ci, i = 1..r-1 (lane-parallel)
    const uint32_t c0 = cols[0];
    uint64_t part = 0;
    for (uint32_t j = lane; j + 1 < geo.r; j += 32) {
      const uint32_t b = c0 ^ cols[j + 1];
      part |= (uint64_t)b << ((j * geo.delta) & 63u);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) part |= __shfl_xor_sync(0xffffffffu, part, o);
    const uint32_t ip = (uint32_t)part;
    bool ok = true;
    for (uint32_t j = lane; j + 1 < geo.r; j += 32) {
      const uint32_t b = c0 ^ cols[j + 1];
      if ((shr32(ip, j * geo.delta) & geo.col_mask) != b) ok = false;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (ok) {
      const uint32_t h0 = ((uint32_t)s_row0[0][ip & 0xff] ^ s_row0[1][(ip >> 8) & 0xff] ^
                           s_row0[2][(ip >> 16) & 0xff] ^ s_row0[3][ip >> 24]) &
                          geo.col_mask;
      ok = (h0 == c0);
    }
    uint32_t rk = 0;
    if (ok) {
      for (uint32_t b = lane; b < geo.eta; b += 32) {
        uint32_t m = 0xffffffffu;
        for (uint32_t row = 0; row < geo.r; ++row) {
          const uint32_t s = stamps[((uint64_t)row << geo.q | cols[row]) * geo.eta + b];
          m = s < m ? s : m;
        }
        rk += m > thr;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
      ok = rk >= cutoff;
    }
    if (accepted && lane == 0) accepted[t] = ok ? 1 : 0;
    if (ok && lane == 0) {
      const unsigned long long pos = atomicAdd(counter, 1ull);
      out_idx[pos] = (uint32_t)t;
      out_cip[pos] = ip;
      out_rk[pos] = rk;
    }
  }
}

// ---------------------------------------------------------------------------
// Element-wise helpers.

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

__global__ void __launch_bounds__(256) merge_kernel(const MergeSrc* __restrict__ srcs, uint32_t nsrc,
                                                    uint64_t n, uint32_t now_common, int take_max,
                                                    uint32_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t acc = rebase(srcs[0].p[i], now_common, srcs[0].lag);
    for (uint32_t g = 1; g < nsrc; ++g) {
      const uint32_t v = rebase(srcs[g].p[i], now_common, srcs[g].lag);
      acc = take_max ? (v > acc ? v : acc) : (v < acc ? v : acc);
    }
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

}  // namespace sspd_dev
