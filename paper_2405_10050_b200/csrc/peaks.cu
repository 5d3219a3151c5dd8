// FP64 / FP32 FMA throughput probes: the roofline denominators for the
// RayCast kernels (MEASURED_PEAKS.json carries only HBM and bf16 figures).
#include "common.cuh"

namespace {

template <typename T, int CHAINS>
__global__ void __launch_bounds__(256) k_fma_probe(T* out, int iters, T b, T c) {
  T a[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) a[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) a[i] = fma(a[i], b, c);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += a[i];
  if (s == (T)-1.2345) out[0] = s;  // keep the chains live
}

// Legacy warp tensor path (mma.sync m16n8k8 tf32, SASS HMMA.1688): 8
// independent accumulators per warp; the tensor-core screen's denominator.
__global__ void __launch_bounds__(256) k_mma_probe(float* out, int iters) {
  const unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[0] = s;
}

}  // namespace

// Launch `blocks` x 256 threads.  dtype 0 = fp64 / 1 = fp32 FMA chains
// (flops = 2 * 8 * iters * blocks * 256); dtype 2 = tf32 mma.sync m16n8k8,
// 8 per warp and iteration (flops = 2 * 16 * 8 * 8 * 8 * 8 * iters * blocks).
extern "C" int vr_fma_probe(int dtype, int blocks, int iters, void* scratch, void* stream) {
  if (blocks <= 0 || iters <= 0 || !scratch) return VR_EINVAL;
  if (dtype == 0)
    k_fma_probe<double, 8><<<blocks, 256, 0, as_stream(stream)>>>((double*)scratch, iters,
                                                                   0.999999, 1e-7);
  else if (dtype == 1)
    k_fma_probe<float, 8><<<blocks, 256, 0, as_stream(stream)>>>((float*)scratch, iters,
                                                                  0.999999f, 1e-7f);
  else if (dtype == 2)
    k_mma_probe<<<blocks, 256, 0, as_stream(stream)>>>((float*)scratch, iters);
  else
    return VR_EINVAL;
  VR_RETURN_LAUNCH();
}
