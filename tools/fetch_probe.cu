// L2 fetch-granularity probe: does cudaLimitMaxL2FetchGranularity change the
// random-access rate of the scan's access patterns?  Each "packet" makes 5
// random 4-byte accesses into a grid of G words (the r recorders of a pair);
// patterns: red.max (fire and forget), atom.max (returning, the window-ring
// path), ld.ca + red.max (the duplicate filter's probe then the stamp).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/fetch_probe tools/fetch_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__);               \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <int MODE>
__global__ void __launch_bounds__(256) access5(size_t n, uint32_t* grid, uint64_t words, uint32_t val,
                                               uint32_t salt, uint32_t* sink) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = mix(i * 0x9e3779b97f4a7c15ULL + salt);
    uint32_t* p[5];
    uint32_t cur[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) p[j] = grid + mix(h + j * 0x9e3779b97f4a7c15ULL) % words;
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 5; ++j) asm volatile("red.global.max.u32 [%0], %1;" ::"l"(p[j]), "r"(val) : "memory");
    } else if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 5; ++j) acc += atomicMax(p[j], val);
    } else if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < 5; ++j) cur[j] = __ldca(p[j]);
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (cur[j] != val) asm volatile("red.global.max.u32 [%0], %1;" ::"l"(p[j]), "r"(val) : "memory");
    } else if (MODE == 3) {  // L2 prefetch, then red
#pragma unroll
      for (int j = 0; j < 5; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(p[j]));
#pragma unroll
      for (int j = 0; j < 5; ++j) asm volatile("red.global.max.u32 [%0], %1;" ::"l"(p[j]), "r"(val) : "memory");
    } else if (MODE == 4) {  // load through L2 only, then red
#pragma unroll
      for (int j = 0; j < 5; ++j) cur[j] = __ldcg(p[j]);
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (cur[j] != val) asm volatile("red.global.max.u32 [%0], %1;" ::"l"(p[j]), "r"(val) : "memory");
    } else if (MODE == 5) {  // load, then returning atomic (the window-ring path)
#pragma unroll
      for (int j = 0; j < 5; ++j) cur[j] = __ldcg(p[j]);
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (cur[j] != val) acc += atomicMax(p[j], val);
    } else if (MODE == 6) {  // L2 prefetch, then returning atomic
#pragma unroll
      for (int j = 0; j < 5; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(p[j]));
#pragma unroll
      for (int j = 0; j < 5; ++j) acc += atomicMax(p[j], val);
    } else if (MODE == 8) {  // packed-bf16 max atomic, returning (the 16-bit narrow scan)
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        unsigned short a, b;
        asm volatile("atom.global.max.noftz.v2.bf16 {%0, %1}, [%2], {%3, %4};"
                     : "=h"(a), "=h"(b)
                     : "l"(p[j]), "h"((unsigned short)(val & 0x7f7f)), "h"((unsigned short)0)
                     : "memory");
        acc += a + b;
      }
    } else {  // loads only (the read half alone)
#pragma unroll
      for (int j = 0; j < 5; ++j) acc += __ldcg(p[j]);
    }
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

template <int MODE>
float run(size_t n, uint32_t* grid, uint64_t words, uint32_t* sink, int blocks) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int w = 0; w < 2; ++w) access5<MODE><<<blocks, 256>>>(n, grid, words, 7 + w, w, sink);
  CK(cudaEventRecord(e0));
  const int reps = 5;
  for (int w = 0; w < reps; ++w) access5<MODE><<<blocks, 256>>>(n, grid, words, 100 + w, 10 + w, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

int main() {
  CK(cudaSetDevice(0));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  size_t dflt = 0;
  CK(cudaDeviceGetLimit(&dflt, cudaLimitMaxL2FetchGranularity));
  printf("device %s, default cudaLimitMaxL2FetchGranularity = %zu B\n", prop.name, dflt);
  const size_t n = 20u << 20;  // packets per launch
  uint32_t* sink;
  CK(cudaMalloc(&sink, 4));
  for (uint64_t mb : {640ull, 10240ull, 40960ull, 81920ull}) {
    const uint64_t words = mb << 18;
    uint32_t* grid;
    if (cudaMalloc(&grid, words * 4) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    CK(cudaMemset(grid, 0, words * 4));
    for (int bpsm : {4, 8, 16}) {
      const int blocks = prop.multiProcessorCount * bpsm;
      printf("grid %6llu MB blocks/SM %2d:", (unsigned long long)mb, bpsm);
      printf(" red %.2f", n / run<0>(n, grid, words, sink, blocks) / 1e6);
      printf(" | atom %.2f", n / run<1>(n, grid, words, sink, blocks) / 1e6);
      printf(" | ld.ca+red %.2f", n / run<2>(n, grid, words, sink, blocks) / 1e6);
      printf(" | pf+red %.2f", n / run<3>(n, grid, words, sink, blocks) / 1e6);
      printf(" | ld.cg+red %.2f", n / run<4>(n, grid, words, sink, blocks) / 1e6);
      printf(" | ld.cg+atom %.2f", n / run<5>(n, grid, words, sink, blocks) / 1e6);
      printf(" | pf+atom %.2f", n / run<6>(n, grid, words, sink, blocks) / 1e6);
      printf(" | ld only %.2f", n / run<7>(n, grid, words, sink, blocks) / 1e6);
      printf(" | bf16x2 atom %.2f Gpkt/s\n", n / run<8>(n, grid, words, sink, blocks) / 1e6);
    }
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, dflt));
    CK(cudaFree(grid));
  }
  return 0;
}
