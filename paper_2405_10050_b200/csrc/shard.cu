// Owner-sharded traversal helpers: row ownership, the
// send order of an all-to-all, its inverse, and the open test from the
// per-vertex edge counts the edge owners return.  Protocol: see
// include/voronray_b200.h ("Owner-sharded traversal") and parallel.py.
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

// Owner of a sorted generator tuple: the high bits of a 64-bit mix, so the
// owner does not correlate with the low bits a rank's own table probes from.
__device__ __forceinline__ uint32_t owner_of(const int32_t* row, int k, int parts) {
  uint64_t h = 0x2545F4914F6CDD1Dull;
  for (int i = 0; i < k; ++i) {
    h ^= (uint32_t)row[i];
    h *= 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
  }
  h *= 0xBF58476D1CE4E5B9ull;
  return (uint32_t)((h >> 32) % (uint64_t)parts);
}

__global__ void k_owner(const int32_t* __restrict__ rows, int64_t n, int k, int parts,
                        uint32_t* __restrict__ owner, int32_t* __restrict__ iota,
                        unsigned long long* __restrict__ counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t o = owner_of(rows + i * k, k, parts);
    owner[i] = o;
    iota[i] = (int32_t)i;
    atomicAdd(counts + o, 1ull);
  }
}

__global__ void k_gather_rows(const int32_t* __restrict__ rows, int k,
                              const int32_t* __restrict__ perm, int64_t n,
                              int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k, c = i - r * k;
    out[i] = rows[(int64_t)perm[r] * k + c];
  }
}

__global__ void k_scatter_rows(const int32_t* __restrict__ rows, int k,
                               const int32_t* __restrict__ perm, int64_t n,
                               int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * k;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / k, c = i - r * k;
    out[(int64_t)perm[r] * k + c] = rows[i];
  }
}

__global__ void k_open_from_counts(const int32_t* __restrict__ cnt, int64_t n_v, int d1,
                                   uint8_t* __restrict__ open_mask,
                                   int32_t* __restrict__ open_count) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_v;
       v += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int k = 0; k < d1; ++k) {
      const bool open = cnt[v * d1 + k] < 2;  // graph.py:127-128
      open_mask[v * d1 + k] = open ? 1 : 0;
      c += open;
    }
    open_count[v] = c;
  }
}

__global__ void k_widen32(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

}  // namespace

extern "C" int vr_shard_bucket(const int32_t* rows, int64_t n, int k, int n_parts, int32_t* perm,
                               int64_t* counts, void* workspace, int64_t* workspace_bytes,
                               void* stream) {
  if (!workspace_bytes || n < 0 || n >= ((int64_t)1 << 31) || k < 1 || n_parts < 1)
    return VR_EINVAL;
  int bits = 1;
  while ((1 << bits) < n_parts) ++bits;
  size_t tmp = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const uint32_t*)nullptr,
                                                  (uint32_t*)nullptr, (const int32_t*)nullptr,
                                                  (int32_t*)nullptr, (int)(n > 0 ? n : 1), 0,
                                                  bits);
  if (e != cudaSuccess) return vr_cuda_status(e);
  const size_t o_own = 0, o_own2 = align256(4 * n), o_iota = o_own2 + align256(4 * n),
               o_tmp = o_iota + align256(4 * n), need = o_tmp + tmp;
  if (!workspace) {
    *workspace_bytes = (int64_t)need;
    return VR_OK;
  }
  if (*workspace_bytes < (int64_t)need) return VR_ECAPACITY;
  if (!counts) return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  if ((e = cudaMemsetAsync(counts, 0, 8 * (size_t)n_parts, st)) != cudaSuccess)
    return vr_cuda_status(e);
  if (n == 0) return VR_OK;
  if (!rows || !perm) return VR_EINVAL;
  char* W = static_cast<char*>(workspace);
  uint32_t* own = reinterpret_cast<uint32_t*>(W + o_own);
  uint32_t* own2 = reinterpret_cast<uint32_t*>(W + o_own2);
  int32_t* iota = reinterpret_cast<int32_t*>(W + o_iota);
  k_owner<<<grid_for(n), 256, 0, st>>>(rows, n, k, n_parts, own, iota,
                                       reinterpret_cast<unsigned long long*>(counts));
  size_t t = tmp;
  e = cub::DeviceRadixSort::SortPairs(W + o_tmp, t, own, own2, iota, perm, (int)n, 0, bits, st);
  return e == cudaSuccess ? VR_OK : vr_cuda_status(e);
}

extern "C" int vr_shard_gather_rows(const int32_t* rows, int k, const int32_t* perm, int64_t n,
                                    int32_t* out, void* stream) {
  if (n <= 0) return VR_OK;
  if (!rows || !perm || !out || k < 1) return VR_EINVAL;
  k_gather_rows<<<grid_for(n * k), 256, 0, as_stream(stream)>>>(rows, k, perm, n, out);
  VR_RETURN_LAUNCH();
}

extern "C" int vr_shard_scatter_rows(const int32_t* rows, int k, const int32_t* perm, int64_t n,
                                     int32_t* out, void* stream) {
  if (n <= 0) return VR_OK;
  if (!rows || !perm || !out || k < 1) return VR_EINVAL;
  k_scatter_rows<<<grid_for(n * k), 256, 0, as_stream(stream)>>>(rows, k, perm, n, out);
  VR_RETURN_LAUNCH();
}

extern "C" int vr_shard_open(const int32_t* edge_counts, int64_t n_v, int d, uint8_t* open_mask,
                             int32_t* open_count, int64_t* open_off, int64_t* n_rays_out,
                             void* workspace, int64_t* workspace_bytes, void* stream) {
  if (!workspace_bytes || n_v < 0 || n_v >= ((int64_t)1 << 31)) return VR_EINVAL;
  size_t tmp = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int64_t*)nullptr,
                                                (int64_t*)nullptr, (int)(n_v > 0 ? n_v : 1));
  if (e != cudaSuccess) return vr_cuda_status(e);
  if (!workspace) {
    *workspace_bytes = (int64_t)tmp;
    return VR_OK;
  }
  if (*workspace_bytes < (int64_t)tmp) return VR_ECAPACITY;
  if (!n_rays_out) return VR_EINVAL;
  *n_rays_out = 0;
  if (n_v == 0) return VR_OK;
  if (!edge_counts || !open_mask || !open_count || !open_off) return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  k_open_from_counts<<<grid_for(n_v), 256, 0, st>>>(edge_counts, n_v, d + 1, open_mask,
                                                    open_count);
  k_widen32<<<grid_for(n_v), 256, 0, st>>>(open_count, open_off, n_v);
  size_t t = tmp;
  if ((e = cub::DeviceScan::ExclusiveSum(workspace, t, open_off, open_off, (int)n_v, st)) !=
      cudaSuccess)
    return vr_cuda_status(e);
  int64_t last = 0;
  int32_t cnt = 0;
  if ((e = cudaMemcpyAsync(&last, open_off + n_v - 1, 8, cudaMemcpyDeviceToHost, st)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(&cnt, open_count + n_v - 1, 4, cudaMemcpyDeviceToHost, st)) !=
          cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return vr_cuda_status(e);
  *n_rays_out = last + cnt;
  return VR_OK;
}
