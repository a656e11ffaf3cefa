// Die probe: (1) which SMs share an L2 partition (die) -- each SM times a
// chain of dependent atomics on one address; the SMs on the address's home
// die are faster -- and (2) whether a table probed by each die's SMs only in
// its own half stays L2-resident to a larger size than one probed by every
// SM everywhere (each L2 partition caches the lines its own SMs read, so a
// table read from both dies may be held twice).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/die_probe tools/die_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t e = (x);                                        \
    if (e != cudaSuccess) {                                     \
      printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); \
      exit(1);                                                  \
    }                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smid() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

// one CTA per SM (big shared allocation); thread 0 times 256 dependent atomics
__global__ void atom_latency(unsigned* target, unsigned long long* out, unsigned zero) {
  extern __shared__ char pad[];
  if (threadIdx.x) return;
  pad[0] = 0;
  unsigned v = 0;
  // warm
  // each atomic's address depends on the previous result (zero is 0 at run time)
  for (int i = 0; i < 8; ++i) v = atomicAdd(target + (v & zero), 1u);
  const long long t0 = clock64();
  for (int i = 0; i < 256; ++i) v = atomicAdd(target + (v & zero), 1u);
  const long long t1 = clock64();
  out[blockIdx.x] = ((unsigned long long)smid() << 48) | (unsigned long long)((t1 - t0) / 256) | ((v & zero) ? 1ull : 0ull);
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// random 16 B loads into `buckets` 16 B buckets; PART: a thread on die d only
// loads buckets of half d
template <int PART>
__global__ void __launch_bounds__(256) probe(const uint4* table, uint64_t buckets, size_t n, const uint8_t* die_of,
                                             unsigned salt, unsigned* sink) {
  const uint32_t d = PART ? die_of[smid()] : 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  const uint64_t half = buckets / 2;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h = mix(i * 0x9e3779b97f4a7c15ULL + salt);
    const uint64_t b = PART ? d * half + h % half : h % buckets;
    uint4 v;
    asm volatile("ld.global.ca.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(table + b));
    acc += v.x ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned* targets;
  CK(cudaMalloc(&targets, 64ull << 20));
  CK(cudaMemset(targets, 0, 64ull << 20));
  unsigned long long* out;
  CK(cudaMalloc(&out, sms * 8));
  CK(cudaFuncSetAttribute(atom_latency, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int naddr = 8;
  std::vector<std::vector<int>> lat(naddr, std::vector<int>(sms, 0));
  for (int a = 0; a < naddr; ++a) {
    unsigned* t = targets + (size_t)a * (1u << 20) + 32 * a;  // 4 MiB apart
    atom_latency<<<sms, 32, 200 * 1024>>>(t, out, 0u);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(sms);
    CK(cudaMemcpy(h.data(), out, sms * 8, cudaMemcpyDeviceToHost));
    for (auto x : h) lat[a][(int)(x >> 48) % sms] = (int)(x & 0xffffffffull);
  }
  // classify by address 0: fast = below the midpoint of min and max
  std::vector<uint8_t> die(sms, 0);
  int lo = 1 << 30, hi = 0;
  for (int s = 0; s < sms; ++s) lo = std::min(lo, lat[0][s]), hi = std::max(hi, lat[0][s]);
  for (int s = 0; s < sms; ++s) die[s] = lat[0][s] > (lo + hi) / 2;
  printf("atomic latency (cycles) per smid for %d addresses; die = slow for address 0 (lo %d hi %d)\n", naddr, lo, hi);
  int n1 = 0;
  for (int s = 0; s < sms; ++s) {
    printf("sm %3d die %d:", s, die[s]);
    for (int a = 0; a < naddr; ++a) printf(" %4d", lat[a][s]);
    printf("\n");
    n1 += die[s];
  }
  // agreement of each address's fast/slow split with address 0's
  for (int a = 1; a < naddr; ++a) {
    int l2 = 1 << 30, h2 = 0, same = 0;
    for (int s = 0; s < sms; ++s) l2 = std::min(l2, lat[a][s]), h2 = std::max(h2, lat[a][s]);
    for (int s = 0; s < sms; ++s) same += (lat[a][s] > (l2 + h2) / 2) == die[s];
    printf("address %d: split agrees with address 0 on %d of %d SMs (or its complement: %d)\n", a, same, sms,
           sms - same);
  }
  printf("die 1 has %d SMs, die 0 has %d\n", n1, sms - n1);

  // (2) partitioned vs unpartitioned probes; a wrong split (smid parity) as control
  uint8_t *d_die, *d_par;
  CK(cudaMalloc(&d_die, sms));
  CK(cudaMalloc(&d_par, sms));
  CK(cudaMemcpy(d_die, die.data(), sms, cudaMemcpyHostToDevice));
  std::vector<uint8_t> par(sms);
  for (int s = 0; s < sms; ++s) par[s] = s & 1;
  CK(cudaMemcpy(d_par, par.data(), sms, cudaMemcpyHostToDevice));
  uint4* table;
  const uint64_t max_mb = 256;
  CK(cudaMalloc(&table, max_mb << 20));
  CK(cudaMemset(table, 0, max_mb << 20));
  unsigned* sink;
  CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const size_t n = 100000000;
  for (uint64_t mb : {32, 48, 64, 80, 96, 112, 128, 160, 192, 256}) {
    const uint64_t buckets = (mb << 20) / 16;
    float best[3] = {1e30f, 1e30f, 1e30f};
    for (int rep = 0; rep < 4; ++rep) {
      for (int mode = 0; mode < 3; ++mode) {
        CK(cudaEventRecord(e0));
        if (mode == 0) probe<0><<<sms * 8, 256>>>(table, buckets, n, d_die, rep, sink);
        else probe<1><<<sms * 8, 256>>>(table, buckets, n, mode == 1 ? d_die : d_par, rep, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep && ms < best[mode]) best[mode] = ms;
      }
    }
    printf("table %4llu MiB: all SMs everywhere %.1f G probes/s | per-die halves %.1f | smid-parity halves %.1f\n",
           (unsigned long long)mb, n / best[0] / 1e6, n / best[1] / 1e6, n / best[2] / 1e6);
  }
  return 0;
}
