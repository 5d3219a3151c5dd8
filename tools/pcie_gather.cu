// Microbenchmark for the e2e design question "can the rays be gathered into
// the kernel's processing order on the way in?": 1e6 rays of x (6 f64) +
// u (6 f64) in pinned host memory, a random permutation;
//   (1) bulk cudaMemcpyAsync H2D of both arrays (the current pipeline's copy),
//   (2) a device kernel gathering rows by the permutation straight from the
//       pinned (UVA-mapped) host arrays,
//   (3) host threads gathering rows into a pinned staging buffer (memcpy),
//   (4) host threads scattering 61-B result rows back to caller order.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pcie_gather tools/pcie_gather.cu -lpthread
#include <cuda_runtime.h>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int D = 6;

__global__ void k_gather(const double* __restrict__ hx, const double* __restrict__ hu,
                         const int* __restrict__ perm, double* __restrict__ dx,
                         double* __restrict__ du, int n) {
  // one thread per (ray, 16-B piece): 3 pieces of x, 3 of u
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * 6) return;
  int i = (int)(t / 6), p = (int)(t % 6);
  int src = perm[i];
  const double2* s = reinterpret_cast<const double2*>((p < 3 ? hx : hu) + (int64_t)src * D) + (p % 3);
  double2* d = reinterpret_cast<double2*>((p < 3 ? dx : du) + (int64_t)i * D) + (p % 3);
  *d = *s;
}

int main(int argc, char** argv) {
  const int n = 1000000;
  const int nth = argc > 1 ? atoi(argv[1]) : (int)std::thread::hardware_concurrency();
  double *hx, *hu, *dx, *du;
  int *hperm, *dperm;
  CK(cudaHostAlloc(&hx, n * D * 8, 0));
  CK(cudaHostAlloc(&hu, n * D * 8, 0));
  CK(cudaHostAlloc(&hperm, n * 4, 0));
  CK(cudaMalloc(&dx, n * D * 8));
  CK(cudaMalloc(&du, n * D * 8));
  CK(cudaMalloc(&dperm, n * 4));
  for (int64_t i = 0; i < (int64_t)n * D; ++i) hx[i] = hu[i] = (double)i;
  std::iota(hperm, hperm + n, 0);
  std::shuffle(hperm, hperm + n, std::mt19937(1));
  CK(cudaMemcpy(dperm, hperm, n * 4, cudaMemcpyHostToDevice));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, s);
    cudaMemcpyAsync(dx, hx, n * D * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(du, hu, n * D * 8, cudaMemcpyHostToDevice, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("bulk H2D 96 MB: %.3f ms (%.1f GB/s)\n", ms, 96e-3 / ms * 1e3 / 1e3 * 1e3 / 1e3);
  }
  for (int grid : {148, 296, 592, 1184, 100000}) {
    for (int rep = 0; rep < 2; ++rep) {
      int64_t nt = (int64_t)n * 6;
      int blocks = grid == 100000 ? (int)((nt + 255) / 256) : grid;
      cudaEventRecord(e0, s);
      if (grid == 100000) {
        k_gather<<<blocks, 256, 0, s>>>(hx, hu, dperm, dx, du, n);
      } else {
        // grid-stride variant via multiple launches of slices
        int per = (n + 7) / 8;
        for (int c = 0; c < 8; ++c) {
          int m = std::min(per, n - c * per);
          k_gather<<<std::min(blocks, (int)((m * 6LL + 255) / 256)), 256, 0, s>>>(
              hx, hu, dperm + c * per, dx + (int64_t)c * per * D, du + (int64_t)c * per * D, m);
        }
      }
      cudaEventRecord(e1, s);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("zero-copy gather (grid %d): %.3f ms (%.1f GB/s useful)\n", grid, ms, 96.0 / ms);
    }
  }
  // host gather into pinned staging
  double* stage;
  CK(cudaHostAlloc(&stage, (size_t)n * 2 * D * 8, 0));
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int w = 0; w < nth; ++w)
      th.emplace_back([&, w] {
        int lo = (int)((int64_t)n * w / nth), hi = (int)((int64_t)n * (w + 1) / nth);
        for (int i = lo; i < hi; ++i) {
          int src = hperm[i];
          memcpy(stage + (int64_t)i * 2 * D, hx + (int64_t)src * D, D * 8);
          memcpy(stage + (int64_t)i * 2 * D + D, hu + (int64_t)src * D, D * 8);
        }
      });
    for (auto& t : th) t.join();
    double el = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    printf("host gather %d threads: %.3f ms (%.1f GB/s)\n", nth, el, 96.0 / el);
  }
  // host scatter of results (idx 4, t 8, rp 48, flag 1) from sorted staging
  int* oidx = (int*)malloc(n * 4);
  double* ot = (double*)malloc(n * 8);
  double* orp = (double*)malloc((size_t)n * D * 8);
  unsigned char* ofl = (unsigned char*)malloc(n);
  int* sidx;
  double *st_, *srp;
  unsigned char* sfl;
  CK(cudaHostAlloc(&sidx, n * 4, 0));
  CK(cudaHostAlloc(&st_, n * 8, 0));
  CK(cudaHostAlloc(&srp, (size_t)n * D * 8, 0));
  CK(cudaHostAlloc(&sfl, n, 0));
  memset(oidx, 0, n * 4); memset(ot, 0, n * 8); memset(orp, 0, (size_t)n * D * 8); memset(ofl, 0, n);
  memset(sidx, 1, n * 4); memset(st_, 1, n * 8); memset(srp, 1, (size_t)n * D * 8); memset(sfl, 1, n);
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int w = 0; w < nth; ++w)
      th.emplace_back([&, w] {
        int lo = (int)((int64_t)n * w / nth), hi = (int)((int64_t)n * (w + 1) / nth);
        for (int i = lo; i < hi; ++i) {
          int dst = hperm[i];
          oidx[dst] = sidx[i];
          ot[dst] = st_[i];
          memcpy(orp + (int64_t)dst * D, srp + (int64_t)i * D, D * 8);
          ofl[dst] = sfl[i];
        }
      });
    for (auto& t : th) t.join();
    double el = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    printf("host scatter %d threads: %.3f ms (%.1f GB/s)\n", nth, el, 61.0 / el);
  }
  return 0;
}
