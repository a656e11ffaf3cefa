// Bare CUDA process cost on a box: context creation, then a 640 MiB alloc + fill (tools/exp_cli_fixed.sh).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
int main() {
  auto t0 = std::chrono::steady_clock::now();
  cudaFree(0);
  auto t1 = std::chrono::steady_clock::now();
  void* p; cudaMalloc(&p, 640u << 20); cudaMemset(p, 0xff, 640u << 20); cudaDeviceSynchronize();
  auto t2 = std::chrono::steady_clock::now();
  printf("context init %.1f ms, 640 MiB alloc+fill %.1f ms\n",
         std::chrono::duration<double, std::milli>(t1 - t0).count(),
         std::chrono::duration<double, std::milli>(t2 - t1).count());
}
