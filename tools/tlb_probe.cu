// Address-footprint probe: does the random-atomic rate of the C2 scan's
// stamp pattern depend on how much of the 80 GiB table a launch touches?
// (profiles/r01_access_probe.txt: ld/atom rates fall ~40% from a 40 GiB to
// an 80 GiB grid.)  One 80 GiB allocation; each "packet" makes 5 returning
// atomicMax accesses, access j inside row region j (16 GiB each, like the
// stamps of rows 0..4 at q16 eta65536), restricted to a part of each row:
//   frac 1/1: the whole row (today's scan, 80 GiB footprint)
//   frac 1/2, 1/4: the first half / quarter of every row (a column-range pass)
// plus single-region spans (all 5 accesses in one contiguous span).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/tlb_probe tools/tlb_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t e = (x);                                        \
    if (e != cudaSuccess) {                                     \
      printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); \
      exit(1);                                                  \
    }                                                           \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// access j goes to region_base + j * region_stride + (random % span)
template <int ATOM>
__global__ void __launch_bounds__(256) access5(size_t n, uint32_t* grid, uint64_t region_stride, uint64_t span,
                                               uint32_t val, uint32_t salt, uint32_t* sink) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = mix(i * 0x9e3779b97f4a7c15ULL + salt);
    uint32_t* p[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) p[j] = grid + j * region_stride + mix(h + j * 0x9e3779b97f4a7c15ULL) % span;
    if (ATOM == 1) {
#pragma unroll
      for (int j = 0; j < 5; ++j) acc += atomicMax(p[j], val);
    } else if (ATOM == 2) {  // load through L2, then the returning atomic (hits the filled line)
      uint32_t cur[5];
#pragma unroll
      for (int j = 0; j < 5; ++j) cur[j] = __ldcg(p[j]);
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (cur[j] != val) acc += atomicMax(p[j], val);
    } else {
#pragma unroll
      for (int j = 0; j < 5; ++j) acc += __ldcg(p[j]);
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  const uint64_t total_words = 80ull << 28;  // 80 GiB of u32
  const uint64_t row_words = 16ull << 28;    // 16 GiB per row region
  uint32_t* grid = nullptr;
  uint32_t* sink = nullptr;
  CK(cudaMalloc(&grid, total_words * 4));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(grid, 0, total_words * 4));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n = 20000000;  // packets per launch (1e8 accesses)
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  struct Case {
    const char* name;
    uint64_t stride, span;
  } cases[] = {
      {"5 rows x 16 GiB (80 GiB, today)", row_words, row_words},
      {"5 rows x 8 GiB  (first half of each row, 40 GiB)", row_words, row_words / 2},
      {"5 rows x 4 GiB  (first quarter of each row, 20 GiB)", row_words, row_words / 4},
      {"one span 80 GiB", 0, total_words},
      {"one span 40 GiB", 0, total_words / 2},
      {"one span 20 GiB", 0, total_words / 4},
  };
  uint32_t launch = 0;  // every launch stores a new, larger value, so ld+atom always issues its atomics
  for (int atom = 0; atom < 3; ++atom) {
    for (const Case& c : cases) {
      for (int bps : {8, 16, 32}) {
        const unsigned blocks = sms * bps;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          CK(cudaEventRecord(a));
          if (atom == 2)
            access5<2><<<blocks, 256>>>(n, grid, c.stride, c.span, ++launch, 1234 + rep, sink);
          else if (atom == 1)
            access5<1><<<blocks, 256>>>(n, grid, c.stride, c.span, ++launch, 1234 + rep, sink);
          else
            access5<0><<<blocks, 256>>>(n, grid, c.stride, c.span, ++launch, 1234 + rep, sink);
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, a, b));
          if (rep && ms < best) best = ms;
        }
        printf("%-7s %-52s blocks/SM %2d: %.3f ms  %.2f G accesses/s\n", atom == 2 ? "ld+atom" : atom ? "atom" : "ld",
               c.name, bps, best,
               5.0 * n / best / 1e6);
      }
    }
  }
  return 0;
}
