// Random-sector scatter microbenchmark: the "random-access roofline" for the
// scan. Each "packet" reads 8 B of input and performs R random
// 4-byte writes into a grid of G words. No hashing: addresses come from a
// cheap mix of the packet index. Modes: 0 = st.global, 1 = red.max, 2 = atom.max
// (returning), 3 = st.global with L2 evict_first hint.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <int MODE, int R>
__global__ void __launch_bounds__(256) scatter(const uint2* __restrict__ in, size_t n, uint32_t* grid,
                                               uint64_t words, uint32_t val, uint32_t* sink) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint2 p = __ldg(in + i);
    uint64_t h = mix(((uint64_t)p.x << 32) | p.y);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      uint64_t a = (mix(h + j * 0x9e3779b97f4a7c15ULL)) % words;
      uint32_t* ptr = grid + a;
      if (MODE == 0) {
        asm volatile("st.global.u32 [%0], %1;" :: "l"(ptr), "r"(val) : "memory");
      } else if (MODE == 1) {
        asm volatile("red.global.max.u32 [%0], %1;" :: "l"(ptr), "r"(val) : "memory");
      } else if (MODE == 2) {
        acc += atomicMax(ptr, val);
      } else {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" :: "l"(ptr), "r"(val), "l"(pol) : "memory");
      }
    }
  }
  if (MODE == 2 && acc == 0xdeadbeef) *sink = acc;
}

__global__ void fill_in(uint2* in, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t h = mix(i * 0x9e3779b97f4a7c15ULL + 12345);
    in[i] = make_uint2((uint32_t)h, (uint32_t)(h >> 32));
  }
}

__global__ void copyk(const uint4* __restrict__ a, uint4* b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

template <int MODE>
float run(const uint2* in, size_t n, uint32_t* grid, uint64_t words, uint32_t* sink, int blocks) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int w = 0; w < 2; ++w) scatter<MODE, 5><<<blocks, 256>>>(in, n, grid, words, 7 + w, sink);
  CK(cudaEventRecord(e0));
  const int reps = 5;
  for (int w = 0; w < reps; ++w) scatter<MODE, 5><<<blocks, 256>>>(in, n, grid, words, 100 + w, sink);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d L2 %d MB\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize >> 20);
  size_t n = 100u << 20;  // 100M packets
  uint2* in; CK(cudaMalloc(&in, n * 8)); uint32_t* sink; CK(cudaMalloc(&sink, 4));
  fill_in<<<1184, 256>>>(in, n);
  uint64_t sizes_mb[] = {16, 64, 640, 10240, 81920};
  for (uint64_t mb : sizes_mb) {
    uint64_t words = mb << 18;
    uint32_t* grid; if (cudaMalloc(&grid, words * 4) != cudaSuccess) { printf("alloc %llu MB failed\n", (unsigned long long)mb); cudaGetLastError(); continue; }
    CK(cudaMemset(grid, 0, words * 4));
    for (int bpsm : {4, 8, 16}) {
      int blocks = prop.multiProcessorCount * bpsm;
      float t0 = run<0>(in, n, grid, words, sink, blocks);
      float t1 = run<1>(in, n, grid, words, sink, blocks);
      float t2 = run<2>(in, n, grid, words, sink, blocks);
      float t3 = run<3>(in, n, grid, words, sink, blocks);
      printf("grid %6llu MB blocks/SM %2d: st %.2f Gpkt/s | red.max %.2f | atom.max %.2f | st.evict_first %.2f  (ms st %.3f)\n",
             (unsigned long long)mb, bpsm, n / t0 / 1e6, n / t1 / 1e6, n / t2 / 1e6, n / t3 / 1e6, t0);
    }
    CK(cudaFree(grid));
  }
  // streaming copy for reference
  size_t cb = 4ull << 30; uint4 *a, *b; CK(cudaMalloc(&a, cb)); CK(cudaMalloc(&b, cb));
  CK(cudaMemset(a, 1, cb));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  copyk<<<148 * 8, 256>>>(a, b, cb / 16);
  CK(cudaEventRecord(e0)); for (int i = 0; i < 5; ++i) copyk<<<148 * 8, 256>>>(a, b, cb / 16);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("copy kernel: %.1f GB/s (read+write)\n", 2.0 * cb * 5 / ms / 1e6);
  CK(cudaDeviceSynchronize());
  return 0;
}
