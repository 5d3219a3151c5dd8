// Random-access ceiling of HBM for the traversal's hash-table kernels
// (k_bump_new / k_open_edges / k_claim touch random 32-B sectors of tables far
// larger than L2): independent random 32-B reads over a table of TABLE_GB, at
// full occupancy, (1) one sector per access, (2) a read of one sector plus an
// atomicAdd on a second random word (the shape of an edge-count bump: key row
// + counter), (3) a streaming read of the same table for the sequential
// figure.  Prints sectors/s and the GB/s ncu's dram__bytes would report
// (32 B per sector read; an atomic is a read-modify-write of its sector).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/rap tools/random_access_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t h) {
  h ^= h >> 33; h *= 0xFF51AFD7ED558CCDull; h ^= h >> 33; h *= 0xC4CEB9FE1A85EC53ull;
  return h ^ (h >> 33);
}

// each thread: `per` dependent-free random sector reads (the address does not
// depend on the loaded data; the compiler keeps several in flight)
__global__ void k_random(const uint4* __restrict__ tab, uint64_t sectors, int per,
                         unsigned long long* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < per; ++i) {
    const uint64_t s = mix(t * 1315423911ull + i) % sectors;
    const uint4 a = __ldcg(tab + 2 * s);
    const uint4 b = __ldcg(tab + 2 * s + 1);
    acc ^= a.x ^ b.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// dependent chain: the next address depends on the loaded value (a probe
// sequence), one sector in flight per thread
__global__ void k_random_dep(const uint4* __restrict__ tab, uint64_t sectors, int per,
                             unsigned long long* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t s = mix(t) % sectors;
  uint32_t acc = 0;
  for (int i = 0; i < per; ++i) {
    const uint4 a = __ldcg(tab + 2 * s);
    acc ^= a.x;
    s = mix(s + a.x + i) % sectors;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_bump(const uint4* __restrict__ tab, int* __restrict__ cnt, uint64_t sectors,
                       uint64_t words, int per, unsigned long long* sink) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < per; ++i) {
    const uint64_t h = mix(t * 1315423911ull + i);
    const uint4 a = __ldcg(tab + 2 * (h % sectors));
    acc ^= a.x;
    atomicAdd(cnt + (h >> 7) % words, 1);
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_stream(const uint4* __restrict__ tab, uint64_t n16, unsigned long long* sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x)
    acc ^= __ldcg(tab + i).x;
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 32.0;
  const uint64_t bytes = (uint64_t)(gb * (1ull << 30));
  const uint64_t sectors = bytes / 32, words = (1ull << 30);
  uint4* tab; int* cnt; unsigned long long* sink;
  CK(cudaMalloc(&tab, bytes));
  CK(cudaMalloc(&cnt, words * 4));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(tab, 1, bytes));
  CK(cudaMemset(cnt, 0, words * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int per = 16;
  const uint64_t threads = 148ull * 2048 * 64;  // many waves at full occupancy
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_random<<<(unsigned)(threads / 256), 256>>>(tab, sectors, per, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("random 32-B reads, independent (two 16-B loads per sector): %.1f G sectors/s = %.0f GB/s (table %.0f GB)\n",
                    threads * per / ms / 1e6, threads * per * 32.0 / ms / 1e6, gb);
    cudaEventRecord(e0);
    k_random_dep<<<(unsigned)(threads / 256), 256>>>(tab, sectors, per, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("random 32-B reads, dependent chain (one in flight per thread): %.1f G sectors/s = %.0f GB/s\n",
                    threads * per / ms / 1e6, threads * per * 32.0 / ms / 1e6);
    cudaEventRecord(e0);
    k_bump<<<(unsigned)(threads / 256), 256>>>(tab, cnt, sectors, words, per, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("random read + random atomicAdd: %.1f G bumps/s = %.0f GB/s of dram traffic (32 B read + 64 B atomic RMW)\n",
                    threads * per / ms / 1e6, threads * per * 96.0 / ms / 1e6);
    cudaEventRecord(e0);
    k_stream<<<148 * 16, 256>>>(tab, bytes / 16, sink);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("streaming read: %.0f GB/s\n", bytes / ms / 1e6);
  }
  return 0;
}
