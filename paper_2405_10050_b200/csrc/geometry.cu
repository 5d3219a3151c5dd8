// Generator packing, filtered nearest neighbour, vertex verification,
// circumcentres and vertex edge directions (include/voronray_b200.h).
#include "common.cuh"

namespace {

template <int D>
__global__ void k_pack(const double* __restrict__ pts, int64_t n, double* __restrict__ rec,
                       unsigned long long* __restrict__ sqmax) {
  constexpr int S = rec_stride(D);
  double local = 0.0;
  const int64_t rows = rec_rows(n);
  for (int64_t i = n + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {  // sentinel rows
#pragma unroll
    for (int k = 0; k < S; ++k) rec[i * S + k] = (k == D) ? CUDART_INF : 0.0;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double sq = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double v = pts[i * D + k];
      rec[i * S + k] = v;
      sq = fma(v, v, sq);
    }
    rec[i * S + D] = sq;
#pragma unroll
    for (int k = D + 1; k < S; ++k) rec[i * S + k] = 0.0;
    local = fmax(local, sq);
  }
  // non-negative doubles order like their bit patterns
  for (int off = 16; off > 0; off >>= 1) local = fmax(local, __shfl_xor_sync(0xffffffffu, local, off));
  if ((threadIdx.x & 31) == 0 && sqmax) atomicMax(sqmax, (unsigned long long)__double_as_longlong(local));
}

// Nearest / second nearest by the expanded squared distance with the
// smallest index on ties (core.py:81-90, 131-142); clean distances after.
template <int D>
__global__ void k_nearest(const double* __restrict__ rec, int64_t n, const double* __restrict__ q,
                          int64_t nq, const uint8_t* __restrict__ skip, int32_t* out_idx,
                          double* out_d1, double* out_d2) {
  constexpr int S = rec_stride(D);
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nq) return;
  double qq[D];
#pragma unroll
  for (int j = 0; j < D; ++j) qq[j] = q[k * D + j];
  double b1 = CUDART_INF, b2 = CUDART_INF;
  int i1 = -1, i2 = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (skip && skip[i]) continue;
    const double* x = rec + i * S;
    double p = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) p = fma(qq[j], x[j], p);
    const double d2 = fma(-2.0, p, x[D]);
    if (d2 < b1) { b2 = b1; i2 = i1; b1 = d2; i1 = (int)i; }
    else if (d2 < b2) { b2 = d2; i2 = (int)i; }
  }
  out_idx[k] = i1;
  auto clean = [&](int i) {
    if (i < 0) return CUDART_INF;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) { const double a = rec[(int64_t)i * S + j] - qq[j]; s = fma(a, a, s); }
    return sqrt(s);
  };
  if (out_d1) out_d1[k] = clean(i1);
  if (out_d2) out_d2[k] = clean(i2);
}

// verify_vertex (core.py:279-296) for a batch of vertices.
template <int D>
__global__ void k_verify(const double* __restrict__ rec, int64_t n, const int32_t* __restrict__ sigma,
                         const double* __restrict__ r, int64_t nv, double tol, uint8_t* ok) {
  constexpr int S = rec_stride(D);
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  double rr[D];
#pragma unroll
  for (int j = 0; j < D; ++j) rr[j] = r[v * D + j];
  int sig[D + 1];
  bool good = true;
#pragma unroll
  for (int a = 0; a <= D; ++a) {
    sig[a] = sigma[v * (D + 1) + a];
    if (sig[a] < 0 || sig[a] >= n) good = false;
  }
#pragma unroll
  for (int a = 0; a <= D; ++a)
#pragma unroll
    for (int b = a + 1; b <= D; ++b)
      if (sig[a] == sig[b]) good = false;
  if (!good) { ok[v] = 0; return; }
  auto dist = [&](int64_t i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) { const double a = rec[i * S + j] - rr[j]; s = fma(a, a, s); }
    return sqrt(s);
  };
  const double rad = dist(sig[0]);
  double dev = 0.0;
#pragma unroll
  for (int a = 1; a <= D; ++a) dev = fmax(dev, fabs(dist(sig[a]) - rad));
  if (!(rad > 0.0) || dev > tol * rad) { ok[v] = 0; return; }
  double mn = CUDART_INF;
  for (int64_t i = 0; i < n; ++i) {
    bool own = false;
#pragma unroll
    for (int a = 0; a <= D; ++a) own |= (sig[a] == i);
    if (!own) mn = fmin(mn, dist(i));
  }
  ok[v] = (mn >= rad * (1.0 - tol)) ? 1 : 0;
}

template <int D>
__global__ void k_circumcenters(const double* __restrict__ rec, const int32_t* __restrict__ sigma,
                                int64_t nv, double* out_r, uint8_t* out_ok) {
  constexpr int S = rec_stride(D);
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const double* x0 = rec + (int64_t)sigma[v * (D + 1)] * S;
  double A[D][D], b[D];
  int piv[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double* xa = rec + (int64_t)sigma[v * (D + 1) + a + 1] * S;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double e = xa[j] - x0[j];
      A[a][j] = 2.0 * e;
      s = fma(e, e, s);
    }
    b[a] = s;
  }
  const bool ok = lu_factor<D>(A, piv);
  if (ok) lu_solve<D>(A, piv, b);
#pragma unroll
  for (int j = 0; j < D; ++j) out_r[v * D + j] = ok ? x0[j] + b[j] : CUDART_NAN;
  if (out_ok) out_ok[v] = ok ? 1 : 0;
}

// _vertex_directions (raycast.py:345-378): rows of D are x_s - x_s0.
template <int D>
__device__ void vertex_dirs(const double* __restrict__ rec, const int32_t* sig, double* out_u,
                            uint8_t* out_ok) {
  constexpr int S = rec_stride(D);
  const double* x0 = rec + (int64_t)sig[0] * S;
  double A[D][D];
  int piv[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double* xa = rec + (int64_t)sig[a + 1] * S;
#pragma unroll
    for (int j = 0; j < D; ++j) A[a][j] = xa[j] - x0[j];
  }
  const bool ok = lu_factor<D>(A, piv);
  for (int k = 0; k <= D; ++k) {
    double v[D];
#pragma unroll
    for (int j = 0; j < D; ++j) v[j] = (k == 0) ? 1.0 : (j == k - 1 ? 1.0 : 0.0);
    bool good = ok;
    if (ok) lu_solve<D>(A, piv, v);
    const double sgn = (k == 0) ? 1.0 : -1.0;
    double nn = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) nn = fma(v[j], v[j], nn);
    const double nrm = sqrt(nn);
    good = good && nrm > 0.0 && isfinite(nrm);
#pragma unroll
    for (int j = 0; j < D; ++j) out_u[k * D + j] = good ? sgn * v[j] / nrm : CUDART_NAN;
    if (out_ok) out_ok[k] = good ? 1 : 0;
  }
}

template <int D>
__global__ void k_vertex_dirs(const double* __restrict__ rec, const int32_t* __restrict__ sigma,
                              int64_t nv, double* out_u, uint8_t* out_ok) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  vertex_dirs<D>(rec, sigma + v * (D + 1), out_u + v * (D + 1) * D,
                 out_ok ? out_ok + v * (D + 1) : nullptr);
}

template <int D>
__global__ void k_pack32(const double* __restrict__ rec, int64_t rows, const double* __restrict__ c0,
                         float* __restrict__ rec32) {
  constexpr int S = rec_stride(D);
  constexpr int S32 = rec32_stride(D);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool sentinel = isinf(rec[i * S + D]);
    double sq = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double v = rec[i * S + k] - c0[k];
      rec32[i * S32 + k] = sentinel ? 0.0f : (float)v;
      sq = fma(v, v, sq);
    }
    rec32[i * S32 + D] = sentinel ? CUDART_INF_F : (float)sq;
#pragma unroll
    for (int k = D + 1; k < S32; ++k) rec32[i * S32 + k] = 0.0f;
  }
}

// fp32 records -> pair-interleaved layout (rows is even: a multiple of 512).
template <int D>
__global__ void k_pairs32(const float* __restrict__ rec32, int64_t rows, float* __restrict__ out) {
  constexpr int S32 = rec32_stride(D);
  constexpr int P2 = rec32p_stride(D);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < rows / 2;
       p += (int64_t)gridDim.x * blockDim.x) {
    const float* a = rec32 + (2 * p) * S32;
    const float* b = a + S32;
    float* o = out + p * P2;
#pragma unroll
    for (int k = 0; k <= D; ++k) {
      o[2 * k] = a[k];
      o[2 * k + 1] = b[k];
    }
#pragma unroll
    for (int k = 2 * D + 2; k < P2; ++k) o[k] = 0.0f;
  }
}

// fp32 records -> mma.sync m16n8k8 B fragments (tf32, round to nearest):
// thread (tile, block, k-step, lane) writes the two values lane l of that
// block and k-step needs; KS = ceil((D + 2) / 8) k8 steps.
template <int D>
__global__ void k_pack_mma(const float* __restrict__ rec32, int64_t rows, float* __restrict__ out) {
  constexpr int KS = (D + 2 + 7) / 8;
  constexpr int S32 = rec32_stride(D);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < rows * 4 * KS;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(q & 31);
    const int step = (int)((q >> 5) % KS);
    const int64_t blk = (q >> 5) / KS;                 // tile * 8 + block
    const int64_t row = blk * 8 + (lane >> 2);
    const float* a = rec32 + row * S32;
    float v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 8 * step + (lane & 3) + 4 * h;
      float f = k < D ? a[k] : (k == D ? a[D] : (k == D + 1 ? 1.0f : 0.0f));
      if (k == D && isinf(f)) f = 1e30f;  // sentinel: never passes (finite, no inf - inf)
      uint32_t t;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(f));
      v[h] = __uint_as_float(t);
    }
    reinterpret_cast<float2*>(out)[q] = make_float2(v[0], v[1]);
  }
}

// fp32 records -> the tcgen05 operand: the same tf32 features as k_pack_mma,
// candidate c of tile t, feature f = 8s + 4q + e at float
// t * 512 KS + s * 512 + ((c & 63) >> 3) * 64 + q * 32 + (c & 7) * 4 + e.
template <int D>
__global__ void k_pack_umma(const float* __restrict__ rec32, int64_t rows, float* __restrict__ out) {
  constexpr int KS = (D + 2 + 7) / 8;
  constexpr int S32 = rec32_stride(D);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * 8 * KS;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / (8 * KS);
    const int f = (int)(i - row * 8 * KS);
    const float* a = rec32 + row * S32;
    float v = f < D ? a[f] : (f == D ? a[D] : (f == D + 1 ? 1.0f : 0.0f));
    if (f == D && isinf(v)) v = 1e30f;  // sentinel: never passes
    uint32_t tb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(tb) : "f"(v));
    const int64_t t = row >> 6;
    const int c = (int)(row & 63), s = f >> 3, q = (f >> 2) & 1, e = f & 3;
    out[t * 512 * KS + s * 512 + (c >> 3) * 64 + q * 32 + (c & 7) * 4 + e] = __uint_as_float(tb);
  }
}

// Descent directions (graph.py:46-85, raycast.py:295-317): per start, the
// two-pass modified Gram-Schmidt basis of the rows x_sigma[i] - x_sigma[0]
// (i = 1 .. k-1, the reference's _orthonormal_rows) and the component of the
// drawn normal z orthogonal to it (two passes, _project_out), one thread per
// start.  bad = the rows are affinely dependent (|v| < tol max(|v0|, 1)).
template <int D>
__global__ void k_descent_dirs(const double* __restrict__ rec, const int32_t* __restrict__ sigma,
                               const int32_t* __restrict__ kcount, const double* __restrict__ z,
                               int64_t n, double tol, double* __restrict__ out_v,
                               double* __restrict__ out_nrm, uint8_t* __restrict__ out_bad) {
  constexpr int S = rec_stride(D);
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int k = kcount[s];
  const int32_t* sg = sigma + s * (D + 1);
  const double* x0 = rec + (int64_t)sg[0] * S;
  double q[D][D];  // orthonormal rows 0 .. k-2
  bool bad = false;
  for (int j = 0; j + 1 < k; ++j) {
    const double* xa = rec + (int64_t)sg[j + 1] * S;
    double v[D];
    double n0 = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      v[c] = xa[c] - x0[c];
      n0 += v[c] * v[c];
    }
    n0 = sqrt(n0);
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < j; ++i) {
        double dot = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) dot += q[i][c] * v[c];
#pragma unroll
        for (int c = 0; c < D; ++c) v[c] -= dot * q[i][c];
      }
    double nv = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) nv += v[c] * v[c];
    nv = sqrt(nv);
    if (nv < tol * fmax(n0, 1.0)) bad = true;
#pragma unroll
    for (int c = 0; c < D; ++c) q[j][c] = v[c] / nv;
  }
  double w[D];
#pragma unroll
  for (int c = 0; c < D; ++c) w[c] = z[s * D + c];
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i + 1 < k; ++i) {
      double dot = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) dot += q[i][c] * w[c];
#pragma unroll
      for (int c = 0; c < D; ++c) w[c] -= dot * q[i][c];
    }
  double nw = 0.0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    nw += w[c] * w[c];
    out_v[s * D + c] = w[c];
  }
  out_nrm[s] = sqrt(nw);
  out_bad[s] = bad ? 1 : 0;
}

inline unsigned blocks_for(int64_t n, int nt) { return (unsigned)((n + nt - 1) / nt); }

}  // namespace

extern "C" int64_t vr_record_rows(int64_t n) { return rec_rows(n); }

extern "C" int vr_pack_generators(const double* pts, int64_t n, int d, double* rec,
                                  double* sqmax_out, void* stream) {
  if (!pts || !rec || n <= 0) return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  if (sqmax_out) {
    cudaError_t e = cudaMemsetAsync(sqmax_out, 0, sizeof(double), st);
    if (e != cudaSuccess) return vr_cuda_status(e);
  }
  const unsigned nb = blocks_for(n, 256) < 4096 ? blocks_for(n, 256) : 4096;
  VR_DISPATCH_D_ALL(d, {
    k_pack<D><<<nb, 256, 0, st>>>(pts, n, rec, reinterpret_cast<unsigned long long*>(sqmax_out));
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_pack_records32(const double* rec, int64_t rows, int d, const double* center,
                                 float* rec32, void* stream) {
  if (!rec || !rec32 || !center || rows <= 0) return VR_EINVAL;
  const unsigned nbk = blocks_for(rows, 256) < 4096 ? blocks_for(rows, 256) : 4096;
  VR_DISPATCH_D(d, {
    k_pack32<D><<<nbk, 256, 0, as_stream(stream)>>>(rec, rows, center, rec32);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_pack_records32_pairs(const float* rec32, int64_t rows, int d, float* out,
                                       void* stream) {
  if (!rec32 || !out || rows <= 0 || (rows & 1)) return VR_EINVAL;
  const unsigned nbk = blocks_for(rows / 2, 256) < 4096 ? blocks_for(rows / 2, 256) : 4096;
  VR_DISPATCH_D(d, {
    k_pairs32<D><<<nbk, 256, 0, as_stream(stream)>>>(rec32, rows, out);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_pack_records_mma(const float* rec32, int64_t rows, int d, float* out,
                                   void* stream) {
  if (!rec32 || !out || rows <= 0 || (rows & 63)) return VR_EINVAL;
  const int64_t n2 = rows * 4 * ((d + 2 + 7) / 8);
  const unsigned nbk = blocks_for(n2, 256) < 4096 ? blocks_for(n2, 256) : 4096;
  VR_DISPATCH_D(d, {
    k_pack_mma<D><<<nbk, 256, 0, as_stream(stream)>>>(rec32, rows, out);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_nearest_batch(const double* rec, int64_t n_gen, int d, const double* q,
                                int64_t n_q, const uint8_t* skip, int32_t* out_idx,
                                double* out_d1, double* out_d2, void* stream) {
  if (!rec || !q || !out_idx || n_gen <= 0) return VR_EINVAL;
  if (n_q <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    k_nearest<D><<<blocks_for(n_q, 128), 128, 0, as_stream(stream)>>>(rec, n_gen, q, n_q, skip,
                                                                        out_idx, out_d1, out_d2);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_verify_vertices(const double* rec, int64_t n_gen, int d, const int32_t* sigma,
                                  const double* r, int64_t n_v, double tol, uint8_t* out_ok,
                                  void* stream) {
  if (!rec || !sigma || !r || !out_ok) return VR_EINVAL;
  if (n_v <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    k_verify<D><<<blocks_for(n_v, 128), 128, 0, as_stream(stream)>>>(rec, n_gen, sigma, r, n_v,
                                                                       tol, out_ok);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_circumcenters(const double* rec, int d, const int32_t* sigma, int64_t n_v,
                                double* out_r, uint8_t* out_ok, void* stream) {
  if (!rec || !sigma || !out_r) return VR_EINVAL;
  if (n_v <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    k_circumcenters<D><<<blocks_for(n_v, 128), 128, 0, as_stream(stream)>>>(rec, sigma, n_v,
                                                                              out_r, out_ok);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_descent_directions(const double* rec, int d, const int32_t* sigma,
                                     const int32_t* k, const double* z, int64_t n, double tol,
                                     double* out_v, double* out_nrm, uint8_t* out_bad,
                                     void* stream) {
  if (!rec || !sigma || !k || !z || !out_v || !out_nrm || !out_bad) return VR_EINVAL;
  if (n <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    k_descent_dirs<D><<<blocks_for(n, 128), 128, 0, as_stream(stream)>>>(
        rec, sigma, k, z, n, tol, out_v, out_nrm, out_bad);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_vertex_directions(const double* rec, int d, const int32_t* sigma, int64_t n_v,
                                    double* out_u, uint8_t* out_ok, void* stream) {
  if (!rec || !sigma || !out_u) return VR_EINVAL;
  if (n_v <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    k_vertex_dirs<D><<<blocks_for(n_v, 128), 128, 0, as_stream(stream)>>>(rec, sigma, n_v, out_u,
                                                                            out_ok);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_pack_records_umma(const float* rec32, int64_t rows, int d, float* out,
                                    void* stream) {
  if (!rec32 || !out || rows <= 0 || (rows & 63)) return VR_EINVAL;
  const int64_t n2 = rows * 8 * ((d + 2 + 7) / 8);
  const unsigned nbk = blocks_for(n2, 256) < 4096 ? blocks_for(n2, 256) : 4096;
  VR_DISPATCH_D(d, {
    k_pack_umma<D><<<nbk, 256, 0, as_stream(stream)>>>(rec32, rows, out);
  });
  VR_RETURN_LAUNCH();
}
