/* Host-only build of the product's synthetic trace generator
 * (paper_1803_11036_b200/csrc/synth.h), with no CUDA runtime, for the CPU
 * legs of bench.py (--impl reference, cpu_baseline), which feed the compiled
 * reference the same traces the device generator makes.  TEST/BENCH
 * INFRASTRUCTURE: built into oracle/libsynth_host.so; the product never
 * loads it.  Same arithmetic as the device kernel, bit for bit
 * (tests/test_synth.py). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "synth.h"

int sspd_synth_zipf_cdf_host(uint32_t hosts, double exponent, uint64_t* cdf_out) {
  if (hosts == 0) return 1;
  double* acc = (double*)malloc(sizeof(double) * hosts);
  if (!acc) return 4;
  double s = 0;
  for (uint32_t i = 0; i < hosts; ++i) {
    s += pow((double)(i + 1), -exponent);
    acc[i] = s;
  }
  const double scale = 9223372036854775808.0; /* 2^63 */
  for (uint32_t i = 0; i < hosts; ++i) {
    const double v = acc[i] / s * scale;
    cdf_out[i] = v >= scale ? (1ull << 63) : (uint64_t)v;
  }
  cdf_out[hosts - 1] = 1ull << 63;
  free(acc);
  return 0;
}

int sspd_synth_pairs_host(const sspd_synth_params* p, const uint64_t* cdf, uint64_t slot, uint64_t j0,
                          uint64_t n, uint32_t* pairs_out) {
  if (!p || !p->hosts || !p->n_shards || p->shard >= p->n_shards || (p->n_super && !p->super_fanout)) return 1;
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)n; ++i)
    sspd_synth_pair(p, cdf, slot, j0 + (uint64_t)i, &pairs_out[2 * i], &pairs_out[2 * i + 1]);
  return 0;
}

uint32_t sspd_synth_super_cip_host(const sspd_synth_params* p, uint32_t i) { return sspd_super_cip(p, i); }
