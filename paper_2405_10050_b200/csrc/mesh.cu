// Mesh-level array operations on the device: lexicographic ordering of
// generator-tuple rows and the edge-incidence check of verify_mesh
// (reference graph.py:202-245, core.py:200-202).
//
// vr_lex_order:   stable lexicographic order of n rows of k int32 (LSD: k
//                 stable radix sorts of one column each, carrying the row
//                 permutation) -- the order of `sorted(dict)` over sigma /
//                 eta tuples, used to materialise a traversal mesh's edge
//                 table like the reference's dict (Mesh.arrays) and by the
//                 incidence count below.
// vr_edge_incidence: the d-subsets of all vertex sigmas (each vertex is
//                 incident to its d+1 edges, graph.py:115-120), sorted and
//                 run-length counted: distinct edge keys + incidence counts.
// vr_edge_check:  for every recorded edge key, the number of incident
//                 vertices (binary search in the incidence table) -- the
//                 reference's edge-consistency pass compares it with the
//                 recorded count (graph.py:214-229).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace {

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline unsigned grid_for(int64_t n, int nt = 256) {
  int64_t b = (n + nt - 1) / nt;
  if (b < 1) b = 1;
  return (unsigned)(b < 8192 ? b : 8192);
}

__global__ void k_iota(int32_t* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// col[i] = rows[idx[i] * k + c] as an order-preserving unsigned key
__global__ void k_column(const int32_t* __restrict__ rows, int k, int c,
                         const int32_t* __restrict__ idx, int64_t n, uint32_t* __restrict__ col) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    col[i] = (uint32_t)rows[(int64_t)idx[i] * k + c] ^ 0x80000000u;
}

template <int D>
__global__ void k_incidences(const int32_t* __restrict__ sigma, int64_t n_v,
                             int32_t* __restrict__ rows) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_v;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t s[D + 1];
#pragma unroll
    for (int q = 0; q <= D; ++q) s[q] = sigma[v * (D + 1) + q];
#pragma unroll
    for (int k = 0; k <= D; ++k) {
      int32_t* o = rows + (v * (D + 1) + k) * D;
      int w = 0;
#pragma unroll
      for (int q = 0; q <= D; ++q)
        if (q != k) o[w++] = s[q];
    }
  }
}

// head[i] = 1 where sorted row i differs from row i-1
template <int D>
__global__ void k_heads(const int32_t* __restrict__ rows, const int32_t* __restrict__ idx,
                        int64_t n, int32_t* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int h = 1;
    if (i > 0) {
      const int32_t* a = rows + (int64_t)idx[i] * D;
      const int32_t* b = rows + (int64_t)idx[i - 1] * D;
      h = 0;
#pragma unroll
      for (int q = 0; q < D; ++q) h |= a[q] != b[q];
    }
    head[i] = h;
  }
}

// unique rows + run lengths from the inclusive scan of the heads
template <int D>
__global__ void k_runs(const int32_t* __restrict__ rows, const int32_t* __restrict__ idx,
                       const int32_t* __restrict__ head, const int32_t* __restrict__ pos,
                       int64_t n, int32_t* __restrict__ keys, int32_t* __restrict__ counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = pos[i] - 1;
    if (head[i]) {
      const int32_t* a = rows + (int64_t)idx[i] * D;
#pragma unroll
      for (int q = 0; q < D; ++q) keys[(int64_t)u * D + q] = a[q];
    }
    atomicAdd(counts + u, 1);
  }
}

template <int D>
__device__ __forceinline__ int cmp_row(const int32_t* a, const int32_t* b) {
#pragma unroll
  for (int q = 0; q < D; ++q) {
    if (a[q] < b[q]) return -1;
    if (a[q] > b[q]) return 1;
  }
  return 0;
}

template <int D>
__global__ void k_edge_check(const int32_t* __restrict__ inc_keys,
                             const int32_t* __restrict__ inc_counts, int64_t n_inc,
                             const int32_t* __restrict__ ekeys, int64_t n_e,
                             int32_t* __restrict__ incident) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_e;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* x = ekeys + e * D;
    int64_t lo = 0, hi = n_inc;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cmp_row<D>(inc_keys + mid * D, x) < 0) lo = mid + 1; else hi = mid;
    }
    incident[e] = (lo < n_inc && cmp_row<D>(inc_keys + lo * D, x) == 0) ? inc_counts[lo] : 0;
  }
}

size_t lex_tmp_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (int)(n > 0 ? n : 1));
  return t;
}

// workspace: col, col_out, idx_alt (n each) + cub temp
size_t lex_ws_bytes(int64_t n) {
  return align256(4 * n) * 3 + align256(lex_tmp_bytes(n));
}

cudaError_t lex_sort(const int32_t* rows, int64_t n, int k, int32_t* order, void* ws,
                     cudaStream_t st) {
  char* W = static_cast<char*>(ws);
  uint32_t* col = reinterpret_cast<uint32_t*>(W);
  uint32_t* col2 = reinterpret_cast<uint32_t*>(W + align256(4 * n));
  int32_t* alt = reinterpret_cast<int32_t*>(W + 2 * align256(4 * n));
  void* tmp = W + 3 * align256(4 * n);
  const size_t tb = lex_tmp_bytes(n);
  int32_t* cur = order;
  int32_t* nxt = alt;
  k_iota<<<grid_for(n), 256, 0, st>>>(cur, n);
  for (int c = k - 1; c >= 0; --c) {
    k_column<<<grid_for(n), 256, 0, st>>>(rows, k, c, cur, n, col);
    size_t t = tb;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, t, col, col2, cur, nxt, (int)n, 0, 32, st);
    if (e != cudaSuccess) return e;
    int32_t* sw = cur;
    cur = nxt;
    nxt = sw;
  }
  if (cur != order)
    return cudaMemcpyAsync(order, cur, 4 * n, cudaMemcpyDeviceToDevice, st);
  return cudaGetLastError();
}

}  // namespace

extern "C" int vr_lex_order(const int32_t* rows, int64_t n, int k, int32_t* order,
                            void* workspace, int64_t* workspace_bytes, void* stream) {
  if (!workspace_bytes || n < 0 || n >= ((int64_t)1 << 31) || k < 1) return VR_EINVAL;
  const size_t need = lex_ws_bytes(n);
  if (!workspace) {
    *workspace_bytes = (int64_t)need;
    return VR_OK;
  }
  if (*workspace_bytes < (int64_t)need) return VR_ECAPACITY;
  if (n == 0) return VR_OK;
  if (!rows || !order) return VR_EINVAL;
  cudaError_t e = lex_sort(rows, n, k, order, workspace, as_stream(stream));
  return e == cudaSuccess ? VR_OK : vr_cuda_status(e);
}

extern "C" int vr_edge_incidence(const int32_t* sigma, int64_t n_v, int d, int32_t* out_keys,
                                 int32_t* out_counts, int64_t* n_unique_out, void* workspace,
                                 int64_t* workspace_bytes, void* stream) {
  if (!workspace_bytes || n_v < 0) return VR_EINVAL;
  if (d < VR_MIN_D || d > VR_MAX_D_ALL) return VR_EDIM;
  const int64_t n = n_v * (d + 1);
  if (n >= ((int64_t)1 << 31)) return VR_EINVAL;
  size_t scan_tmp = 0;
  cub::DeviceScan::InclusiveSum(nullptr, scan_tmp, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)(n > 0 ? n : 1));
  const size_t o_rows = 0, o_idx = align256(4 * n * d), o_head = o_idx + align256(4 * n),
               o_pos = o_head + align256(4 * n), o_scan = o_pos + align256(4 * n),
               o_lex = o_scan + align256(scan_tmp), need = o_lex + lex_ws_bytes(n);
  if (!workspace) {
    *workspace_bytes = (int64_t)need;
    return VR_OK;
  }
  if (*workspace_bytes < (int64_t)need) return VR_ECAPACITY;
  if (!n_unique_out) return VR_EINVAL;
  *n_unique_out = 0;
  if (n == 0) return VR_OK;
  if (!sigma || !out_keys || !out_counts) return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  char* W = static_cast<char*>(workspace);
  int32_t* rows = reinterpret_cast<int32_t*>(W + o_rows);
  int32_t* idx = reinterpret_cast<int32_t*>(W + o_idx);
  int32_t* head = reinterpret_cast<int32_t*>(W + o_head);
  int32_t* pos = reinterpret_cast<int32_t*>(W + o_pos);
  cudaError_t e;
  VR_DISPATCH_D_ALL(d, { k_incidences<D><<<grid_for(n_v), 256, 0, st>>>(sigma, n_v, rows); });
  if ((e = lex_sort(rows, n, d, idx, W + o_lex, st)) != cudaSuccess) return vr_cuda_status(e);
  VR_DISPATCH_D_ALL(d, { k_heads<D><<<grid_for(n), 256, 0, st>>>(rows, idx, n, head); });
  size_t t = scan_tmp;
  if ((e = cub::DeviceScan::InclusiveSum(W + o_scan, t, head, pos, (int)n, st)) != cudaSuccess)
    return vr_cuda_status(e);
  int32_t nu = 0;
  if ((e = cudaMemcpyAsync(&nu, pos + n - 1, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return vr_cuda_status(e);
  if ((e = cudaMemsetAsync(out_counts, 0, 4 * (size_t)nu, st)) != cudaSuccess)
    return vr_cuda_status(e);
  VR_DISPATCH_D_ALL(d, {
    k_runs<D><<<grid_for(n), 256, 0, st>>>(rows, idx, head, pos, n, out_keys, out_counts);
  });
  *n_unique_out = nu;
  VR_RETURN_LAUNCH();
}

extern "C" int vr_edge_check(const int32_t* inc_keys, const int32_t* inc_counts, int64_t n_inc,
                             const int32_t* edge_keys, int64_t n_e, int d, int32_t* incident,
                             void* stream) {
  if (n_e <= 0) return VR_OK;
  if (!edge_keys || !incident || (n_inc > 0 && (!inc_keys || !inc_counts))) return VR_EINVAL;
  VR_DISPATCH_D_ALL(d, {
    k_edge_check<D><<<grid_for(n_e), 256, 0, as_stream(stream)>>>(inc_keys, inc_counts, n_inc,
                                                                    edge_keys, n_e, incident);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_vertex_edges(const int32_t* sigma, int64_t n_v, int d, int32_t* out,
                               void* stream) {
  if (n_v <= 0) return VR_OK;
  if (!sigma || !out) return VR_EINVAL;
  VR_DISPATCH_D_ALL(d, {
    k_incidences<D><<<grid_for(n_v), 256, 0, as_stream(stream)>>>(sigma, n_v, out);
  });
  VR_RETURN_LAUNCH();
}
