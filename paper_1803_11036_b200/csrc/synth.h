// synth.h -- deterministic synthetic (cip, oip) traces for the C2/C3/C5
// workloads (§8f row f3), identical on host and device.
//
// Mirrors the shape of the reference generator (workload.cpp:215-300):
// Zipf-distributed background hosts that draw opposite hosts from fixed
// per-host pools (so no background host can exceed the pool size), plus
// injected super points -- scanners (one inside host -> many distinct
// targets) and DDoS victims (one inside host <- many distinct sources), which
// after orientation (workload.cpp:146-175) are both a cip with many distinct
// oips.  Unlike the reference's mt19937_64 stream it is counter-based (pair j
// of slot s is a pure function of (seed, s, j)), so any slice can be made on
// the GPU or on host cores independently and bit-identically; Zipf sampling
// uses an integer CDF built once on the host.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SSPD_HD __host__ __device__ __forceinline__
#else
#define SSPD_HD static inline
#endif

typedef struct {
  uint64_t seed;
  uint32_t hosts;           // background hosts (Zipf ranks)
  uint32_t pool;            // distinct opposite hosts per background host; 0 = uniform pairs
  uint32_t n_super;         // injected super points
  uint32_t super_fanout;    // distinct opposite hosts per super point, per slot
  uint64_t pairs_per_slot;  // total pairs per slot, injected ones first
  uint32_t shard;           // router index (C3: disjoint shards per GPU)
  uint32_t n_shards;
} sspd_synth_params;

SSPD_HD uint64_t sspd_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

SSPD_HD uint32_t sspd_super_cip(const sspd_synth_params* p, uint32_t i) {
  return (uint32_t)sspd_mix64(p->seed ^ 0x5ca77e4d0d05ULL ^ ((uint64_t)i << 24));
}

SSPD_HD uint32_t sspd_bg_cip(const sspd_synth_params* p, uint32_t host) {
  return (uint32_t)sspd_mix64(p->seed ^ 0xb6e151628aed2a6bULL ^ ((uint64_t)host << 20));
}

// First index i with cdf[i] > u (cdf ascending, last entry = 2^63).
SSPD_HD uint32_t sspd_zipf_pick(const uint64_t* cdf, uint32_t n, uint64_t u) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (cdf[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Pair j of slot s.  Shards split the background stream: shard t of n keeps
// the packets with j % n == t (C3: each router sees a disjoint share); the
// injected super points are split the same way, so a super point's fan-out
// is only complete in the union of the routers.
SSPD_HD void sspd_synth_pair(const sspd_synth_params* p, const uint64_t* cdf, uint64_t slot,
                             uint64_t j_local, uint32_t* cip, uint32_t* oip) {
  const uint64_t j = j_local * p->n_shards + p->shard;
  const uint64_t injected = (uint64_t)p->n_super * p->super_fanout;
  if (j < injected) {
    const uint32_t i = (uint32_t)(j / p->super_fanout);
    const uint64_t t = j % p->super_fanout;
    *cip = sspd_super_cip(p, i);
    *oip = (uint32_t)sspd_mix64(p->seed ^ 0x1f83d9abfb41bd6bULL ^ ((uint64_t)i << 32) ^ t);
    return;
  }
  const uint64_t h = sspd_mix64(p->seed ^ (slot * 0xd1b54a32d192ed03ULL) ^ (j * 0x9e3779b97f4a7c15ULL));
  if (p->pool == 0) {  // uniform (cip, oip) background (C1)
    *cip = (uint32_t)h;
    *oip = (uint32_t)(h >> 32);
    return;
  }
  const uint32_t host = sspd_zipf_pick(cdf, p->hosts, h >> 1);
  const uint32_t slot_in_pool = (uint32_t)(sspd_mix64(h) % p->pool);
  *cip = sspd_bg_cip(p, host);
  *oip = (uint32_t)sspd_mix64(p->seed ^ 0x3c6ef372fe94f82bULL ^ ((uint64_t)host << 16) ^ slot_in_pool);
}
