// Level-synchronous Voronoi traversal on the device.
//
// Reference: the depth-first, edge-counting traversal voronoi_graph
// (pkg/src/voronray/graph.py:88-146).  Per BFS level the host driver
// (graph.py in this package) runs:
//   open_edges  -> edges sigma\sigma[k] of the frontier with count < 2
//                  (graph.py:127-135), prefix sum
//   emit_rays   -> one LU per frontier vertex, the outward direction of each
//                  open edge (raycast.py:345-378), ray (x=r, u, eta)
//   RayCast     -> the fused kernel of raycast_core.cuh
//   claim       -> sigma' = sorted(eta + {i}); insert-or-find in the vertex
//                  hash set; the smallest ray id wins each new key
//   winners     -> new_flag per ray; prefix sum gives deterministic ids
//   finalize    -> store sigma', fp64 circumcentre, bump the d+1 edge counts
//                  (graph.py:115-120)
//   boundary    -> escaped rays become BoundaryRay(sigma, u) (graph.py:138-139)
// All tables are open-addressed with linear probing; a slot's state goes
// 0 (empty) -> 1 (being written) -> 2 (published) with release/acquire order.
#include <cub/device/device_scan.cuh>

#include "trav_core.cuh"

namespace {

inline unsigned nb(int64_t n, int nt = 256) { return (unsigned)((n + nt - 1) / nt); }

Tables from(const vr_traverse_tables* p) {
  return Tables{p->vkeys, p->vstate, p->vval, p->vlevel, p->vcap,
                p->ekeys, p->estate, p->ecount, p->ecap, p->overflow,
                edge_stride(p->estate, p->ecount)};
}

bool pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

// ---------------------------------------------------------------------------
// Edge-table compaction in two passes over the slot states (vr_trav_edges_*):
// published-slot counts per chunk of EC_CHUNK slots, a cub scan of the chunk
// counts, then each chunk writes its published keys / counts in slot order.
// Same order as flag + prefix sum + k_edge_compact, without the int64 flag
// scan over the whole table (config 5: 2^30 slots, 25 -> ~5 ms).
// ---------------------------------------------------------------------------
constexpr int EC_NT = 256, EC_PER = 16, EC_CHUNK = EC_NT * EC_PER;

__global__ void __launch_bounds__(EC_NT) k_count_published(const int32_t* __restrict__ state,
                                                           int ss, int64_t cap,
                                                           int64_t* __restrict__ chunk_cnt) {
  const int64_t base = (int64_t)blockIdx.x * EC_CHUNK;
  int c = 0;
#pragma unroll
  for (int i = 0; i < EC_PER; ++i) {
    const int64_t h = base + i * EC_NT + threadIdx.x;
    c += (h < cap && state[(int64_t)ss * h] == 2) ? 1 : 0;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  __shared__ int sw[EC_NT / 32];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < EC_NT / 32; ++w) tot += sw[w];
    chunk_cnt[blockIdx.x] = tot;
  }
}

__global__ void __launch_bounds__(EC_NT) k_compact_published(Tables t,
                                                             const int64_t* __restrict__ chunk_off,
                                                             int64_t* __restrict__ out_slot) {
  // thread j owns slots base + j * EC_PER .. + EC_PER (contiguous: slot order
  // = thread order), an exclusive block scan of the per-thread counts
  const int64_t base = (int64_t)blockIdx.x * EC_CHUNK + (int64_t)threadIdx.x * EC_PER;
  unsigned m = 0u;
#pragma unroll
  for (int i = 0; i < EC_PER; ++i) {
    const int64_t h = base + i;
    if (h < t.ecap && t.estate[(int64_t)t.es * h] == 2) m |= 1u << i;
  }
  const int c = __popc(m);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += o;
  }
  __shared__ int sw[EC_NT / 32];
  if (lane == 31) sw[w] = inc;
  __syncthreads();
  int pre = 0;
  for (int k = 0; k < w; ++k) pre += sw[k];
  int64_t o = chunk_off[blockIdx.x] + pre + inc - c;
  while (m) {  // the slot of every output row (4 B); the rows move in k_gather_edges
    const int i = __ffs(m) - 1;
    m &= m - 1;
    out_slot[o++] = base + i;
  }
}

// Output rows in order: coalesced writes, key rows read in increasing slot
// order.
template <int D>
__global__ void k_gather_edges(Tables t, const int64_t* __restrict__ out_slot, int64_t n,
                               int32_t* __restrict__ out_keys, int32_t* __restrict__ out_count) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * (D + 1);
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = q / (D + 1);
    const int a = (int)(q - o * (D + 1));
    const int64_t h = out_slot[o];
    if (a < D) out_keys[o * D + a] = t.ekeys[h * D + a];
    else out_count[o] = t.ecount[(int64_t)t.es * h];
  }
}

}  // namespace

extern "C" int vr_trav_edges_count(const vr_traverse_tables* tab, int64_t* chunk_off,
                                   int64_t* n_edges, void* workspace, int64_t* workspace_bytes,
                                   void* stream) {
  if (!tab || !workspace_bytes) return VR_EINVAL;
  const int64_t nc = (tab->ecap + EC_CHUNK - 1) / EC_CHUNK;
  if (nc >= ((int64_t)1 << 31)) return VR_EINVAL;
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(nc + 1));
  if (!workspace) {
    *workspace_bytes = (int64_t)tmp;
    return VR_OK;
  }
  if (!chunk_off || !n_edges || *workspace_bytes < (int64_t)tmp) return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(chunk_off + nc, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return vr_cuda_status(e);
  k_count_published<<<(unsigned)nc, EC_NT, 0, st>>>(tab->estate,
                                                    edge_stride(tab->estate, tab->ecount),
                                                    tab->ecap, chunk_off);
  if ((e = cudaGetLastError()) != cudaSuccess) return vr_cuda_status(e);
  // in-place exclusive scan over nc + 1 entries: chunk_off[nc] = total
  if ((e = cub::DeviceScan::ExclusiveSum(workspace, tmp, chunk_off, chunk_off, (int)(nc + 1),
                                         st)) != cudaSuccess)
    return vr_cuda_status(e);
  if ((e = cudaMemcpyAsync(n_edges, chunk_off + nc, sizeof(int64_t), cudaMemcpyDeviceToHost,
                           st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return vr_cuda_status(e);
  return VR_OK;
}

extern "C" int vr_trav_edges_compact(const vr_traverse_tables* tab, int d,
                                     const int64_t* chunk_off, int64_t n_edges, int64_t* out_slot,
                                     int32_t* out_keys, int32_t* out_count, void* stream) {
  if (!tab || !chunk_off || !out_slot || !out_keys || !out_count || n_edges < 0) return VR_EINVAL;
  const Tables t = from(tab);
  const int64_t nc = (tab->ecap + EC_CHUNK - 1) / EC_CHUNK;
  cudaStream_t st = as_stream(stream);
  k_compact_published<<<(unsigned)nc, EC_NT, 0, st>>>(t, chunk_off, out_slot);
  if (n_edges == 0) VR_RETURN_LAUNCH();
  VR_DISPATCH_D_ALL(d, {
    const int64_t work = n_edges * (D + 1);
    const unsigned g = (unsigned)((work + 255) / 256 < 148 * 32 ? (work + 255) / 256 : 148 * 32);
    k_gather_edges<D><<<g, 256, 0, st>>>(t, out_slot, n_edges, out_keys, out_count);
  });
  VR_RETURN_LAUNCH();
}

namespace {

}  // namespace

extern "C" int vr_trav_insert_vertices(const vr_traverse_tables* tab, int d, const int32_t* sigma,
                                       int64_t n_v, int32_t base_id, int32_t level,
                                       int bump_edges_flag, void* stream) {
  if (!tab || !sigma || !pow2(tab->vcap) || !pow2(tab->ecap)) return VR_EINVAL;
  if (n_v <= 0) return VR_OK;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_insert_vertices<D><<<nb(n_v), 256, 0, as_stream(stream)>>>(t, sigma, n_v, base_id, level,
                                                                  bump_edges_flag);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_rehash_edges(const vr_traverse_tables* tab, int d, const int32_t* okeys,
                                    const int32_t* ostate, const int32_t* ocount, int64_t ocap,
                                    void* stream) {
  if (!tab || !okeys || !ostate || !ocount || !pow2(tab->ecap)) return VR_EINVAL;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_rehash_edges<D><<<nb(ocap), 256, 0, as_stream(stream)>>>(t, okeys, ostate, ocount, ocap);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_open_edges_sub(const vr_traverse_tables* tab, int d, const int32_t* sigma,
                                      int64_t n_v, int sub_n, int sub_j, uint8_t* open_mask,
                                      int32_t* open_count, void* stream) {
  if (!tab || !sigma || !open_mask || !open_count || sub_n < 1 || sub_j < 0 || sub_j >= sub_n)
    return VR_EINVAL;
  if (n_v <= 0) return VR_OK;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_open_edges<D><<<nb(n_v, 128), 128, 0, as_stream(stream)>>>(t, sigma, n_v, open_mask,
                                                                  open_count, sub_n, sub_j);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_open_edges(const vr_traverse_tables* tab, int d, const int32_t* sigma,
                                  int64_t n_v, uint8_t* open_mask, int32_t* open_count,
                                  void* stream) {
  return vr_trav_open_edges_sub(tab, d, sigma, n_v, 1, 0, open_mask, open_count, stream);
}

extern "C" int vr_trav_emit_rays(const double* rec, int d, const int32_t* sigma, const double* r,
                                 int64_t n_v, const uint8_t* open_mask, const int64_t* open_off,
                                 double* ray_x, double* ray_u, int32_t* ray_eta,
                                 int32_t* ray_parent, int32_t* bad, void* stream) {
  if (!rec || !sigma || !r || !open_mask || !open_off || !ray_x || !ray_u || !ray_eta ||
      !ray_parent || !bad)
    return VR_EINVAL;
  if (n_v <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    k_emit_rays<D><<<nb(n_v, 128), 128, 0, as_stream(stream)>>>(
        rec, sigma, r, n_v, open_mask, open_off, ray_x, ray_u, ray_eta, ray_parent, bad);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_claim(const vr_traverse_tables* tab, int d, const int32_t* ray_eta,
                             const int32_t* hit_idx, const uint8_t* hit_flag, int64_t n_rays,
                             int32_t level, int32_t* out_sigma, int64_t* out_slot,
                             int32_t* new_flag, int32_t* esc_flag, void* stream) {
  if (!tab || !ray_eta || !hit_idx || !hit_flag || !out_sigma || !out_slot || !new_flag ||
      !esc_flag)
    return VR_EINVAL;
  if (n_rays <= 0) return VR_OK;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_claim<D><<<nb(n_rays), 256, 0, as_stream(stream)>>>(t, ray_eta, hit_idx, hit_flag, n_rays,
                                                          level, out_sigma, out_slot);
    k_winners<D><<<nb(n_rays), 256, 0, as_stream(stream)>>>(t, out_slot, hit_flag, n_rays, level,
                                                            new_flag, esc_flag);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_finalize(const vr_traverse_tables* tab, const double* rec, int d,
                                const int32_t* ray_sigma, const int64_t* slot,
                                const int32_t* new_flag, const int64_t* new_off, int64_t n_rays,
                                int32_t base_id, int32_t* vsig, double* vr, int32_t* bad,
                                int bump, void* stream) {
  if (!tab || !rec || !ray_sigma || !slot || !new_flag || !new_off || !vsig || !vr || !bad)
    return VR_EINVAL;
  if (n_rays <= 0) return VR_OK;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_finalize<D><<<nb(n_rays, 128), 128, 0, as_stream(stream)>>>(
        t, rec, ray_sigma, slot, new_flag, new_off, n_rays, base_id, vsig, vr, bad);
    if (bump)
      k_bump_new<D><<<nb(n_rays), 256, 0, as_stream(stream)>>>(t, ray_sigma, new_flag, n_rays);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_boundary(int d, const int32_t* esc_flag, const int64_t* esc_off,
                                const int32_t* ray_parent, const double* ray_u, int64_t n_rays,
                                const int32_t* frontier_sigma, int64_t base_b, int32_t* bsig,
                                double* bu, void* stream) {
  if (!esc_flag || !esc_off || !ray_parent || !ray_u || !frontier_sigma || !bsig || !bu)
    return VR_EINVAL;
  if (n_rays <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    k_boundary<D><<<nb(n_rays), 256, 0, as_stream(stream)>>>(esc_flag, esc_off, ray_parent, ray_u,
                                                             n_rays, frontier_sigma, base_b, bsig,
                                                             bu);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_published(const int32_t* state, int64_t cap, int32_t* flag, void* stream) {
  if (!state || !flag) return VR_EINVAL;
  if (cap <= 0) return VR_OK;
  k_published<<<nb(cap), 256, 0, as_stream(stream)>>>(state, cap, flag);
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_edge_compact(const vr_traverse_tables* tab, int d, const int64_t* off,
                                    int32_t* out_keys, int32_t* out_count, void* stream) {
  if (!tab || !off || !out_keys || !out_count) return VR_EINVAL;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_edge_compact<D><<<nb(t.ecap), 256, 0, as_stream(stream)>>>(t, off, out_keys, out_count);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_claim_sigma(const vr_traverse_tables* tab, int d, const int32_t* rows,
                                   int64_t n, int32_t level, int64_t* out_slot,
                                   int32_t* new_flag, void* stream) {
  if (n <= 0) return VR_OK;
  if (!tab || !rows || !out_slot || !new_flag) return VR_EINVAL;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_claim_sigma<D><<<nb(n), 256, 0, as_stream(stream)>>>(t, rows, n, level, out_slot);
  });
  k_winners_sigma<<<nb(n), 256, 0, as_stream(stream)>>>(t, out_slot, n, level, new_flag);
  VR_RETURN_LAUNCH();
}

extern "C" int vr_trav_bump_keys(const vr_traverse_tables* tab, int d, const int32_t* keys,
                                 int64_t n, int32_t* counts_out, void* stream) {
  if (n <= 0) return VR_OK;
  if (!tab || !keys) return VR_EINVAL;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_bump_keys<D><<<nb(n), 256, 0, as_stream(stream)>>>(t, keys, n);
    if (counts_out)
      k_edge_counts<D><<<nb(n), 256, 0, as_stream(stream)>>>(t, keys, n, counts_out);
  });
  VR_RETURN_LAUNCH();
}
