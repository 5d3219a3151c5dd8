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

}  // namespace

// Launch `blocks` x 256 threads, each doing iters * CHAINS FMAs.
// flops = 2 * 8 * iters * blocks * 256.  dtype: 0 = fp64, 1 = fp32.
extern "C" int vr_fma_probe(int dtype, int blocks, int iters, void* scratch, void* stream) {
  if (blocks <= 0 || iters <= 0 || !scratch) return VR_EINVAL;
  if (dtype == 0)
    k_fma_probe<double, 8><<<blocks, 256, 0, as_stream(stream)>>>((double*)scratch, iters,
                                                                   0.999999, 1e-7);
  else
    k_fma_probe<float, 8><<<blocks, 256, 0, as_stream(stream)>>>((float*)scratch, iters,
                                                                  0.999999f, 1e-7f);
  VR_RETURN_LAUNCH();
}
