// Shared helpers for the sm_100a kernels: status mapping, d-dispatch,
// generator record layout, and the TMA bulk-copy / mbarrier primitives used
// to stage generator tiles into shared memory.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "../../include/voronray_b200.h"

#define VR_MIN_D 2
#define VR_MAX_D 8       // the fp32 / tensor-core / pruned fast paths
#define VR_MAX_D_ALL 16  // exhaustive fp64 RayCast, MC, traversal, mesh ops

// Reference tolerances (pkg/src/voronray/core.py:24-29).
#define VR_TOL_VERTEX 1e-8
#define VR_TOL_DEGENERATE 1e-10
#define VR_HALFSPACE_SLACK 1e-12

// Record arrays hold ceil(n / VR_REC_PAD) * VR_REC_PAD rows; rows >= n are
// sentinels [0, .., 0, +inf] (|x|^2 = inf never passes the RayCast screen).
#define VR_REC_PAD 512
__host__ __device__ constexpr int64_t rec_rows(int64_t n) {
  return (n + VR_REC_PAD - 1) / VR_REC_PAD * VR_REC_PAD;
}

// Doubles per packed generator record: [x_0..x_{d-1}, |x|^2] rounded up to an
// even count so every record starts on a 16-byte boundary (LDS.128 / TMA).
__host__ __device__ constexpr int rec_stride(int d) { return (d + 2) & ~1; }

// Floats per fp32 screening record: [x_0 - c_0 .. x_{d-1} - c_{d-1}, |x - c|^2]
// rounded up to a multiple of 4 (16-B rows).
__host__ __device__ constexpr int rec32_stride(int d) { return (d + 4) & ~3; }

// Floats per PAIR of candidates in the pair-interleaved fp32 layout used by
// the pruned kernel: [x_0a x_0b x_1a x_1b .. x_{d-1}a x_{d-1}b |.|^2_a |.|^2_b]
// rounded up to a multiple of 4, so one LDS.128 feeds two packed FFMA2.
__host__ __device__ constexpr int rec32p_stride(int d) { return (2 * d + 5) & ~3; }

static inline int vr_cuda_status(cudaError_t e) {
  return e == cudaSuccess ? VR_OK : (VR_ECUDA_BASE - (int)e);
}

#define VR_RETURN_LAUNCH()                                  \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    return vr_cuda_status(_e);                              \
  } while (0)

#define VR_DISPATCH_D(d, ...)                               \
  switch (d) {                                              \
    case 2: { constexpr int D = 2; __VA_ARGS__; } break;    \
    case 3: { constexpr int D = 3; __VA_ARGS__; } break;    \
    case 4: { constexpr int D = 4; __VA_ARGS__; } break;    \
    case 5: { constexpr int D = 5; __VA_ARGS__; } break;    \
    case 6: { constexpr int D = 6; __VA_ARGS__; } break;    \
    case 7: { constexpr int D = 7; __VA_ARGS__; } break;    \
    case 8: { constexpr int D = 8; __VA_ARGS__; } break;    \
    default: return VR_EDIM;                                \
  }

// d = 9 .. 16 (the exhaustive fp64 paths only), and d = 2 .. 16.
#define VR_DISPATCH_D_HIGH(d, ...)                           \
  switch (d) {                                               \
    case 9: { constexpr int D = 9; __VA_ARGS__; } break;     \
    case 10: { constexpr int D = 10; __VA_ARGS__; } break;   \
    case 11: { constexpr int D = 11; __VA_ARGS__; } break;   \
    case 12: { constexpr int D = 12; __VA_ARGS__; } break;   \
    case 13: { constexpr int D = 13; __VA_ARGS__; } break;   \
    case 14: { constexpr int D = 14; __VA_ARGS__; } break;   \
    case 15: { constexpr int D = 15; __VA_ARGS__; } break;   \
    case 16: { constexpr int D = 16; __VA_ARGS__; } break;   \
    default: return VR_EDIM;                                 \
  }

#define VR_DISPATCH_D_ALL(d, ...)                            \
  if ((d) > VR_MAX_D) {                                      \
    VR_DISPATCH_D_HIGH(d, __VA_ARGS__)                       \
  } else {                                                   \
    VR_DISPATCH_D(d, __VA_ARGS__)                            \
  }

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// mbarrier + cp.async.bulk (TMA 1-D bulk copy, SASS UBLKCP) primitives.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}

// Global -> shared bulk copy completing on `bar` (bytes multiple of 16).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------------------
// Small fixed-size linear algebra in registers (d <= 8).
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ double dot_seq(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) s = fma(a[k], b[k], s);
  return s;
}

// Partial-pivot LU of a DxD row-major matrix in place; returns false when a
// pivot is exactly zero or non-finite.
template <int D>
__device__ bool lu_factor(double (&A)[D][D], int (&piv)[D]) {
#pragma unroll
  for (int c = 0; c < D; ++c) {
    int p = c;
    double best = fabs(A[c][c]);
#pragma unroll
    for (int r = c + 1; r < D; ++r) {
      double v = fabs(A[r][c]);
      if (v > best) { best = v; p = r; }
    }
    piv[c] = p;
    if (!(best > 0.0) || !isfinite(best)) return false;
    // row swap with static indices only (a runtime row index would put A in
    // local memory): exact, so the factors are unchanged
#pragma unroll
    for (int r = c + 1; r < D; ++r) {
      const bool sw = r == p;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double a = A[c][k], b = A[r][k];
        A[c][k] = sw ? b : a;
        A[r][k] = sw ? a : b;
      }
    }
    double inv = 1.0 / A[c][c];
#pragma unroll
    for (int r = c + 1; r < D; ++r) {
      double f = A[r][c] * inv;
      A[r][c] = f;
#pragma unroll
      for (int k = c + 1; k < D; ++k) A[r][k] = fma(-f, A[c][k], A[r][k]);
    }
  }
  return true;
}

// Solve A x = b with the factors from lu_factor (b overwritten by x).
template <int D>
__device__ void lu_solve(const double (&A)[D][D], const int (&piv)[D], double (&b)[D]) {
  // P b first (full-row swaps in lu_factor give P A = L U), then L y = P b.
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const int p = piv[c];
#pragma unroll
    for (int r = c + 1; r < D; ++r) {
      const bool sw = r == p;
      const double x = b[c], y = b[r];
      b[c] = sw ? y : x;
      b[r] = sw ? x : y;
    }
  }
#pragma unroll
  for (int c = 0; c < D; ++c) {
#pragma unroll
    for (int r = c + 1; r < D; ++r) b[r] = fma(-A[r][c], b[c], b[r]);
  }
#pragma unroll
  for (int c = D - 1; c >= 0; --c) {
    double s = b[c];
#pragma unroll
    for (int k = c + 1; k < D; ++k) s = fma(-A[c][k], b[k], s);
    b[c] = s / A[c][c];
  }
}
