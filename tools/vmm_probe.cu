// Does the physical allocation shape change the random-access rate on an
// 80 GB table?  Same 5-access pattern as fetch_probe.cu on (a) cudaMalloc and
// (b) cuMemCreate chunks mapped into one VA range reserved with a large
// alignment (the driver may then use larger GPU pages).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/vmm_probe tools/vmm_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t e = (x);                                        \
    if (e != cudaSuccess) {                                     \
      printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); \
      exit(1);                                                  \
    }                                                           \
  } while (0)
#define CD(x)                                 \
  do {                                        \
    CUresult r = (x);                         \
    if (r != CUDA_SUCCESS) {                  \
      const char* s;                          \
      cuGetErrorString(r, &s);                \
      printf("CU %s @%d\n", s, __LINE__);     \
      exit(1);                                \
    }                                         \
  } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <int MODE>
__global__ void __launch_bounds__(256) access5(size_t n, uint32_t* grid, uint64_t words, uint32_t val, uint32_t salt,
                                               uint32_t* sink) {
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
      for (int j = 0; j < 5; ++j) acc += atomicMax(p[j], val);
    } else if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 5; ++j) acc += __ldcg(p[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 5; ++j) cur[j] = __ldcg(p[j]);
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (cur[j] != val) acc += atomicMax(p[j], val);
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
  for (int w = 0; w < 5; ++w) access5<MODE><<<blocks, 256>>>(n, grid, words, 100 + w, 10 + w, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / 5;
}

void bench(const char* what, uint32_t* grid, uint64_t words, uint32_t* sink, int sms) {
  const size_t n = 20u << 20;
  CK(cudaMemset(grid, 0, words * 4));
  for (int bpsm : {8, 16}) {
    const int blocks = sms * bpsm;
    printf("%-40s blocks/SM %2d: atom %.2f | ld %.2f | ld+atom %.2f Gpkt/s\n", what, bpsm,
           n / run<0>(n, grid, words, sink, blocks) / 1e6, n / run<1>(n, grid, words, sink, blocks) / 1e6,
           n / run<2>(n, grid, words, sink, blocks) / 1e6);
  }
}

int main() {
  CK(cudaSetDevice(0));
  CD(cuInit(0));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  uint32_t* sink;
  CK(cudaMalloc(&sink, 4));
  const uint64_t bytes = 80ull << 30;
  const uint64_t words = bytes / 4;
  {
    uint32_t* g;
    CK(cudaMalloc(&g, bytes));
    bench("cudaMalloc 80 GiB", g, words, sink, prop.multiProcessorCount);
    CK(cudaFree(g));
  }
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  size_t gmin = 0, grec = 0;
  CD(cuMemGetAllocationGranularity(&gmin, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CD(cuMemGetAllocationGranularity(&grec, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("VMM granularity: minimum %zu B, recommended %zu B\n", gmin, grec);
  for (uint64_t chunk : {2ull << 20, 512ull << 20, 2ull << 30, 16ull << 30}) {
    CUdeviceptr va;
    CD(cuMemAddressReserve(&va, bytes, chunk, 0, 0));
    const uint64_t nchunks = bytes / chunk;
    CUmemGenericAllocationHandle* hs = new CUmemGenericAllocationHandle[nchunks];
    bool ok = true;
    for (uint64_t i = 0; i < nchunks && ok; ++i) {
      if (cuMemCreate(&hs[i], chunk, &ap, 0) != CUDA_SUCCESS) ok = false;
      else CD(cuMemMap(va + i * chunk, chunk, 0, hs[i], 0));
    }
    if (!ok) {
      printf("chunk %llu: cuMemCreate failed\n", (unsigned long long)chunk);
      continue;
    }
    CUmemAccessDesc ad = {};
    ad.location = ap.location;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CD(cuMemSetAccess(va, bytes, &ad, 1));
    char name[64];
    snprintf(name, sizeof name, "VMM 80 GiB, %llu MiB chunks, aligned", (unsigned long long)(chunk >> 20));
    bench(name, reinterpret_cast<uint32_t*>(va), words, sink, prop.multiProcessorCount);
    CD(cuMemUnmap(va, bytes));
    for (uint64_t i = 0; i < nchunks; ++i) CD(cuMemRelease(hs[i]));
    CD(cuMemAddressFree(va, bytes));
    delete[] hs;
  }
  return 0;
}
