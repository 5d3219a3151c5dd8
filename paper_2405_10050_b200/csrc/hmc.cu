// Heuristic Monte-Carlo post-processing on the device (
// reference pkg/src/voronray/integrate_hmc.py:21-91): the pyramid-sum volume
// of a cell from its face areas, the two-term interface rule (vertex mean +
// centroid of the interface's vertices) and the cone rule for cell
// integrals, as segmented reductions over the sigma-keyed vertex set.
//
// Face index (vr_hmc_face_index): every vertex sigma belongs to the
// d(d+1)/2 interfaces (sigma_a, sigma_b), a < b.  The (pair key, vertex id)
// list is radix-sorted (stable, so a face's vertices stay in vertex order --
// the reference's face_vertices order, core.py:223-246), and an interface's
// vertices are the equal-key run found by binary search.  Boundary edges
// (count 1) mark their generators' cells unbounded and their generator pairs
// as unbounded interfaces (core.py:248-276).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline unsigned grid_for(int64_t n, int nt = 256) {
  int64_t b = (n + nt - 1) / nt;
  if (b < 1) b = 1;
  return (unsigned)(b < 8192 ? b : 8192);
}

__host__ __device__ inline uint64_t pair_key(int32_t a, int32_t b) {
  return ((uint64_t)(uint32_t)(a < b ? a : b) << 32) | (uint32_t)(a < b ? b : a);
}

template <int D>
__global__ void k_vertex_pairs(const int32_t* __restrict__ sigma, int64_t n_v,
                               uint64_t* __restrict__ keys, int32_t* __restrict__ vid) {
  constexpr int P = D * (D + 1) / 2;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_v;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t s[D + 1];
#pragma unroll
    for (int k = 0; k <= D; ++k) s[k] = sigma[v * (D + 1) + k];
    int q = 0;
#pragma unroll
    for (int a = 0; a <= D; ++a)
#pragma unroll
      for (int b = a + 1; b <= D; ++b) {
        keys[v * P + q] = pair_key(s[a], s[b]);
        vid[v * P + q] = (int32_t)v;
        ++q;
      }
  }
}

// Boundary edges (count 1): their generators' cells are unbounded, every
// generator pair inside them is an unbounded interface.
template <int D>
__global__ void k_boundary_pairs(const int32_t* __restrict__ ekey,
                                 const int32_t* __restrict__ ecount, int64_t n_e,
                                 uint8_t* __restrict__ cell_unbounded,
                                 uint64_t* __restrict__ ukeys,
                                 unsigned long long* __restrict__ n_ukeys) {
  constexpr int P = D * (D - 1) / 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_e;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (ecount[e] != 1) continue;
    int32_t s[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      s[k] = ekey[e * D + k];
      cell_unbounded[s[k]] = 1;
    }
    const unsigned long long base = atomicAdd(n_ukeys, (unsigned long long)P);
    int q = 0;
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = a + 1; b < D; ++b) ukeys[base + q++] = pair_key(s[a], s[b]);
  }
}

// Distinct mesh neighbours per generator: one count per distinct pair key.
__global__ void k_neighbour_counts(const uint64_t* __restrict__ keys, int64_t n,
                                   int32_t* __restrict__ nb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    if (i > 0 && keys[i - 1] == k) continue;
    atomicAdd(nb + (int32_t)(k >> 32), 1);
    atomicAdd(nb + (int32_t)(uint32_t)k, 1);
  }
}

__device__ __forceinline__ int64_t lower_bound(const uint64_t* a, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Reference built-in integrands (integrands.py:10-44): 1 const, 2 sin(x_1^2),
// 3 linear a.x + b.
template <int D>
__device__ __forceinline__ double integrand(int kind, const double* coef, const double* p) {
  if (kind == 1) return coef[0];
  if (kind == 2) return sin(p[0] * p[0]);
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) v = fma(coef[k], p[k], v);
  return v + coef[D];
}

struct Coef {
  double c[VR_MAX_D_ALL + 1];
};

// Per queried interface (cell i, neighbour j, area A):
//   status 0 ok, 1 unbounded interface, 2 fewer than d vertices, 3 not an
//   interface of the mesh;  count K, vertex mean of f (compensated sum, the
//   reference uses math.fsum), centroid, and
//   F = (d * mean + f(centroid)) * A / (d + 1)   (integrate_hmc.py:42-64).
template <int D>
__global__ void k_hmc_faces(const uint64_t* __restrict__ keys, const int32_t* __restrict__ vid,
                            int64_t n_keys, const uint64_t* __restrict__ ukeys, int64_t n_ukeys,
                            const double* __restrict__ r, const int32_t* __restrict__ fi,
                            const int32_t* __restrict__ fj, const double* __restrict__ area,
                            int64_t n_f, int kind, Coef coef, double* __restrict__ out_F,
                            int32_t* __restrict__ out_status, int32_t* __restrict__ out_first,
                            int32_t* __restrict__ out_count, double* __restrict__ out_mean,
                            double* __restrict__ out_centroid) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n_f;
       f += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = pair_key(fi[f], fj[f]);
    const int64_t lo = lower_bound(keys, n_keys, key);
    int64_t hi = lo;
    while (hi < n_keys && keys[hi] == key) ++hi;
    const int K = (int)(hi - lo);
    out_first[f] = (int32_t)lo;
    out_count[f] = K;
    int status = 0;
    if (K == 0) status = 3;
    else if (n_ukeys > 0) {
      const int64_t u = lower_bound(ukeys, n_ukeys, key);
      if (u < n_ukeys && ukeys[u] == key) status = 1;
    }
    if (status == 0 && K < D) status = 2;
    out_status[f] = status;
    double F = CUDART_NAN, mean = CUDART_NAN;
    double c[D];
#pragma unroll
    for (int k = 0; k < D; ++k) c[k] = CUDART_NAN;
    if (status == 0) {
      // centroid: coordinate sums in vertex order, / K (numpy mean over rows)
      double sum[D];
#pragma unroll
      for (int k = 0; k < D; ++k) sum[k] = 0.0;
      double hs = 0.0, ls = 0.0;  // Neumaier-compensated sum of f(v)
      for (int64_t q = lo; q < hi; ++q) {
        const double* rv = r + (int64_t)vid[q] * D;
        double p[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          p[k] = rv[k];
          sum[k] += p[k];
        }
        if (kind) {
          const double x = integrand<D>(kind, coef.c, p);
          const double t = hs + x;
          ls += fabs(hs) >= fabs(x) ? (hs - t) + x : (x - t) + hs;
          hs = t;
        }
      }
#pragma unroll
      for (int k = 0; k < D; ++k) c[k] = sum[k] / (double)K;
      if (kind) {
        mean = (hs + ls) / (double)K;
        F = ((double)D * mean + integrand<D>(kind, coef.c, c)) * area[f] / (double)(D + 1);
      }
    }
    if (out_F) out_F[f] = F;
    if (out_mean) out_mean[f] = mean;
    if (out_centroid) {
#pragma unroll
      for (int k = 0; k < D; ++k) out_centroid[f * D + k] = c[k];
    }
  }
}

// Per cell c (faces [off[c], off[c+1]) of the CSR, sorted by j):
//   volume = (1/d) sum_j |x_i - x_j| / 2 * A_ij          (integrate_hmc.py:21-39)
//   integral = (d * sum_j h_j F_ij / d + f(x_i) volume) / (d + 1)   (:67-91)
//   status bit 0: unbounded cell, bit 1: a mesh neighbour has no area
//   (MissingNeighbor), bit 2: an interface failed (status of k_hmc_faces).
template <int D>
__global__ void k_hmc_cells(const double* __restrict__ rec, const int32_t* __restrict__ cells,
                            int64_t n_c, const int64_t* __restrict__ off,
                            const int32_t* __restrict__ fj, const double* __restrict__ area,
                            const double* __restrict__ F, const int32_t* __restrict__ fstatus,
                            const uint8_t* __restrict__ cell_unbounded,
                            const int32_t* __restrict__ nb_count, int kind, Coef coef,
                            const double* __restrict__ volume_in, double* __restrict__ out_volume,
                            double* __restrict__ out_integral, int32_t* __restrict__ out_status) {
  constexpr int S = rec_stride(D);
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_c;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = cells[c];
    const double* xi = rec + (int64_t)i * S;
    double vol = 0.0, base = 0.0;
    int found = 0, bad = 0;
    for (int64_t f = off[c]; f < off[c + 1]; ++f) {
      const double* xj = rec + (int64_t)fj[f] * S;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double t = xj[k] - xi[k];
        s += t * t;
      }
      const double h = 0.5 * sqrt(s);
      vol += h * area[f];
      if (fstatus) {
        if (fstatus[f] != 3) ++found;
        if (fstatus[f] != 0) bad = 1;
        if (kind) base += h * F[f] / (double)D;
      }
    }
    vol /= (double)D;
    int st = 0;
    if (cell_unbounded && cell_unbounded[i]) st |= 1;
    if (nb_count && nb_count[i] > found) st |= 2;
    if (bad) st |= 4;
    out_volume[c] = vol;
    if (out_integral) {
      const double v = volume_in ? volume_in[c] : vol;
      double x[D];
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = xi[k];
      out_integral[c] = kind ? ((double)D * base + integrand<D>(kind, coef.c, x) * v) /
                                   (double)(D + 1)
                             : CUDART_NAN;
    }
    out_status[c] = st;
  }
}

struct IndexPlan {
  size_t o_kin, o_vin, o_utmp, o_cnt, o_tmp, tmp, total;
};

int index_plan(int64_t n_v, int d, int64_t n_e, int64_t n_gen, IndexPlan& p) {
  const int64_t P = (int64_t)d * (d + 1) / 2;
  const int64_t U = n_e * (int64_t)d * (d - 1) / 2;
  const int64_t nk = n_v * P;
  if (nk >= ((int64_t)1 << 31) || U >= ((int64_t)1 << 31)) return VR_EINVAL;
  int bits = 1;
  while (bits < 31 && ((int64_t)1 << bits) <= n_gen) ++bits;
  size_t t1 = 0, t2 = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, t1, (const uint64_t*)nullptr,
                                                  (uint64_t*)nullptr, (const int32_t*)nullptr,
                                                  (int32_t*)nullptr, (int)(nk > 0 ? nk : 1), 0,
                                                  32 + bits);
  if (e != cudaSuccess) return vr_cuda_status(e);
  e = cub::DeviceRadixSort::SortKeys(nullptr, t2, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                     (int)(U > 0 ? U : 1), 0, 32 + bits);
  if (e != cudaSuccess) return vr_cuda_status(e);
  p.tmp = t1 > t2 ? t1 : t2;
  p.o_kin = 0;
  p.o_vin = align256(p.o_kin + 8 * nk);
  p.o_utmp = align256(p.o_vin + 4 * nk);
  p.o_cnt = align256(p.o_utmp + 8 * (U > 0 ? U : 1));
  p.o_tmp = align256(p.o_cnt + 8);
  p.total = p.o_tmp + p.tmp;
  return VR_OK;
}

}  // namespace

extern "C" int vr_hmc_face_index(const int32_t* sigma, int64_t n_v, int d, int64_t n_gen,
                                 const int32_t* edge_key, const int32_t* edge_count,
                                 int64_t n_e, uint64_t* keys, int32_t* vid, uint64_t* ukeys,
                                 int64_t* n_ukeys_out, uint8_t* cell_unbounded,
                                 int32_t* nb_count, void* workspace, int64_t* workspace_bytes,
                                 void* stream) {
  if (!workspace_bytes || n_v < 0 || n_e < 0 || n_gen < 1) return VR_EINVAL;
  if (d < VR_MIN_D || d > VR_MAX_D_ALL) return VR_EDIM;
  IndexPlan P;
  int s = index_plan(n_v, d, n_e, n_gen, P);
  if (s) return s;
  if (!workspace) {
    *workspace_bytes = (int64_t)P.total;
    return VR_OK;
  }
  if (*workspace_bytes < (int64_t)P.total) return VR_ECAPACITY;
  if (!sigma || !keys || !vid || !ukeys || !n_ukeys_out || !cell_unbounded || !nb_count ||
      (n_e > 0 && (!edge_key || !edge_count)))
    return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  char* W = static_cast<char*>(workspace);
  uint64_t* kin = reinterpret_cast<uint64_t*>(W + P.o_kin);
  int32_t* vin = reinterpret_cast<int32_t*>(W + P.o_vin);
  uint64_t* utmp = reinterpret_cast<uint64_t*>(W + P.o_utmp);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(W + P.o_cnt);
  void* tmp = W + P.o_tmp;
  const int64_t nk = n_v * (int64_t)d * (d + 1) / 2;
  int bits = 1;
  while (bits < 31 && ((int64_t)1 << bits) <= n_gen) ++bits;
  cudaError_t e;
  if ((e = cudaMemsetAsync(cell_unbounded, 0, n_gen, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(nb_count, 0, 4 * n_gen, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(cnt, 0, 8, st)) != cudaSuccess)
    return vr_cuda_status(e);
  VR_DISPATCH_D_ALL(d, {
    if (nk > 0) k_vertex_pairs<D><<<grid_for(n_v), 256, 0, st>>>(sigma, n_v, kin, vin);
    if (n_e > 0)
      k_boundary_pairs<D><<<grid_for(n_e), 256, 0, st>>>(edge_key, edge_count, n_e,
                                                         cell_unbounded, utmp, cnt);
  });
  size_t t = P.tmp;
  if (nk > 0) {
    if ((e = cub::DeviceRadixSort::SortPairs(tmp, t, kin, keys, vin, vid, (int)nk, 0, 32 + bits,
                                             st)) != cudaSuccess)
      return vr_cuda_status(e);
    k_neighbour_counts<<<grid_for(nk), 256, 0, st>>>(keys, nk, nb_count);
  }
  unsigned long long nu = 0;
  if ((e = cudaMemcpyAsync(&nu, cnt, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return vr_cuda_status(e);
  *n_ukeys_out = (int64_t)nu;
  if (nu > 0) {
    t = P.tmp;
    if ((e = cub::DeviceRadixSort::SortKeys(tmp, t, utmp, ukeys, (int)nu, 0, 32 + bits, st)) !=
        cudaSuccess)
      return vr_cuda_status(e);
  }
  VR_RETURN_LAUNCH();
}

extern "C" int vr_hmc_faces(const uint64_t* keys, const int32_t* vid, int64_t n_keys,
                            const uint64_t* ukeys, int64_t n_ukeys, const double* r, int d,
                            const int32_t* face_i, const int32_t* face_j, const double* area,
                            int64_t n_f, int integrand_kind, const double* coef, double* out_F,
                            int32_t* out_status, int32_t* out_first, int32_t* out_count,
                            double* out_mean, double* out_centroid, void* stream) {
  if (n_f <= 0) return VR_OK;
  if (!keys || !vid || !r || !face_i || !face_j || !out_status || !out_first || !out_count ||
      (integrand_kind && (!area || !coef || !out_F)) || integrand_kind < 0 || integrand_kind > 3)
    return VR_EINVAL;
  Coef c{};
  const int ncoef = integrand_kind == 1 ? 1 : (integrand_kind == 3 ? d + 1 : 0);
  for (int k = 0; k < ncoef; ++k) c.c[k] = coef[k];
  VR_DISPATCH_D_ALL(d, {
    k_hmc_faces<D><<<grid_for(n_f, 128), 128, 0, as_stream(stream)>>>(
        keys, vid, n_keys, ukeys, n_ukeys, r, face_i, face_j, area, n_f, integrand_kind, c,
        out_F, out_status, out_first, out_count, out_mean, out_centroid);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_hmc_cells(const double* rec, int d, const int32_t* cells, int64_t n_c,
                            const int64_t* face_off, const int32_t* face_j, const double* area,
                            const double* F, const int32_t* face_status,
                            const uint8_t* cell_unbounded, const int32_t* nb_count,
                            int integrand_kind, const double* coef, const double* volume_in,
                            double* out_volume, double* out_integral, int32_t* out_status,
                            void* stream) {
  if (n_c <= 0) return VR_OK;
  if (!rec || !cells || !face_off || !face_j || !area || !out_volume || !out_status ||
      integrand_kind < 0 || integrand_kind > 3 || (integrand_kind && (!F || !coef)))
    return VR_EINVAL;
  Coef c{};
  const int ncoef = integrand_kind == 1 ? 1 : (integrand_kind == 3 ? d + 1 : 0);
  for (int k = 0; k < ncoef; ++k) c.c[k] = coef[k];
  VR_DISPATCH_D_ALL(d, {
    k_hmc_cells<D><<<grid_for(n_c, 128), 128, 0, as_stream(stream)>>>(
        rec, cells, n_c, face_off, face_j, area, F, face_status, cell_unbounded, nb_count,
        integrand_kind, c, volume_in, out_volume, out_integral, out_status);
  });
  VR_RETURN_LAUNCH();
}
