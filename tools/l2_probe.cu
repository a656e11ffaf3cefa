// How much of the B200's L2 serves random 16 B probes: random ld.global.cg.v4 loads (the key set's
// bucket loads, L1 bypassed) into a table of S MiB, S from 8 to 256, with and without an
// evict_last L2 policy, after one warm-up pass.  Rate in G loads/s: where it falls off is the
// table size past which probes start to miss L2 (profiles/r02_ab_keyset.md, "L2 reach").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/l2_probe tools/l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_cg_last(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}

template <int HINT>
__global__ void __launch_bounds__(256) probe(const uint4* __restrict__ t, uint64_t n, uint64_t iters,
                                             uint32_t seed, uint32_t* sink) {
  uint64_t pol = 0;
  if (HINT) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  uint64_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + seed;
  uint32_t acc = 0;
  for (uint64_t i = 0; i < iters; i += 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // four independent probes in flight per thread
      x ^= x >> 12; x ^= x << 25; x ^= x >> 27;
      const uint64_t idx = (((x * 0x2545F4914F6CDD1Dull) >> 32) * n) >> 32;  // uniform in [0, n)
      v[u] = HINT ? ld_cg_last(t + idx, pol) : ld_cg(t + idx);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t maxb = 256ull << 20;
  uint4* t;
  uint32_t* sink;
  cudaMalloc(&t, maxb);
  cudaMalloc(&sink, 4);
  cudaMemset(t, 1, maxb);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8;
  const uint64_t iters = 1024;
  const double loads = (double)blocks * 256 * iters;
  printf("random 16 B ld.global.cg probes, %d CTAs x 256 threads x %llu loads\n", blocks, (unsigned long long)iters);
  printf("table MiB | plain G loads/s | evict_last G loads/s\n");
  for (size_t mib : {8, 16, 32, 48, 64, 80, 96, 112, 128, 192, 256}) {
    const uint64_t n = (mib << 20) / 16;
    double rate[2];
    for (int h = 0; h < 2; ++h) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (h) probe<1><<<blocks, 256>>>(t, n, iters, 7 + rep, sink);
        else probe<0><<<blocks, 256>>>(t, n, iters, 7 + rep, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        rate[h] = loads / (ms / 1e3) / 1e9;
      }
    }
    printf("%9zu | %15.1f | %20.1f\n", mib, rate[0], rate[1]);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
  return 0;
}
