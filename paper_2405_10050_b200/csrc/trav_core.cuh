// Device side of the level-synchronous traversal: open-addressed hash
// tables (vertex set keyed by sorted sigma, edge counts keyed by sigma minus
// one generator) and the per-element bodies of the level kernels, shared by
// the per-level kernels (traverse.cu) and the persistent small-level kernel
// (level_small.cu).  Reference: graph.py:88-146.
#pragma once
#include <cuda/atomic>

#include "common.cuh"

namespace {

using dev_atomic = cuda::atomic_ref<int32_t, cuda::thread_scope_device>;

struct Tables {
  int32_t* vkeys;
  int32_t* vstate;
  int32_t* vval;
  int32_t* vlevel;
  int64_t vcap;
  int32_t* ekeys;
  int32_t* estate;
  int32_t* ecount;
  int64_t ecap;
  int32_t* overflow;
  // Stride (in int32) of the edge table's state / count arrays: 2 when they
  // are interleaved as (state, count) pairs -- ecount == estate + 1, so a
  // slot's state and counter share one 32-B sector and a bump costs one
  // random sector less -- else 1 (two separate arrays).
  int es = 1;
};

inline int edge_stride(const int32_t* estate, const int32_t* ecount) {
  return ecount == estate + 1 ? 2 : 1;
}
__device__ __forceinline__ int edge_stride_dev(const int32_t* estate, const int32_t* ecount) {
  return ecount == estate + 1 ? 2 : 1;
}

template <int KW>
__device__ __forceinline__ uint64_t hash_key(const int32_t (&k)[KW]) {
  uint64_t h = 0x9E3779B97F4A7C15ull;
#pragma unroll
  for (int i = 0; i < KW; ++i) {
    h ^= (uint32_t)k[i];
    h *= 0xFF51AFD7ED558CCDull;
    h ^= h >> 32;
  }
  h *= 0xC4CEB9FE1A85EC53ull;
  return h ^ (h >> 29);
}

template <int KW>
__device__ __forceinline__ bool key_eq(const int32_t* slot, const int32_t (&k)[KW]) {
  bool eq = true;
#pragma unroll
  for (int i = 0; i < KW; ++i) eq &= (__ldcg(slot + i) == k[i]);
  return eq;
}

// Insert-or-find.  On insertion `init(slot)` runs before the slot is
// published.  Returns the slot or -1 (table full -> *overflow = 1).
template <int KW, class Init>
__device__ int64_t table_insert(int32_t* keys, int32_t* state, int64_t cap,
                                const int32_t (&k)[KW], bool& inserted, int32_t* overflow,
                                Init init, int ss = 1) {
  const uint64_t mask = (uint64_t)cap - 1;
  uint64_t h = hash_key<KW>(k) & mask;
  inserted = false;
  for (int64_t probe = 0; probe < cap; ++probe) {
    dev_atomic st(state[(int64_t)ss * h]);
    int32_t s = st.load(cuda::memory_order_acquire);
    if (s == 0) {
      int32_t expect = 0;
      if (st.compare_exchange_strong(expect, 1, cuda::memory_order_relaxed)) {
#pragma unroll
        for (int i = 0; i < KW; ++i) keys[h * KW + i] = k[i];
        init((int64_t)h);
        st.store(2, cuda::memory_order_release);
        inserted = true;
        return (int64_t)h;
      }
      s = expect;
    }
    while (s == 1) s = st.load(cuda::memory_order_acquire);
    if (key_eq<KW>(keys + h * KW, k)) return (int64_t)h;
    h = (h + 1) & mask;
  }
  atomicExch(overflow, 1);
  return -1;
}

// Lookup only (no concurrent inserts in the same kernel).
template <int KW>
__device__ int64_t table_find(const int32_t* keys, const int32_t* state, int64_t cap,
                              const int32_t (&k)[KW], int ss = 1) {
  const uint64_t mask = (uint64_t)cap - 1;
  uint64_t h = hash_key<KW>(k) & mask;
  for (int64_t probe = 0; probe < cap; ++probe) {
    const int32_t s = __ldcg(state + (int64_t)ss * h);
    if (s == 0) return -1;
    if (key_eq<KW>(keys + h * KW, k)) return (int64_t)h;
    h = (h + 1) & mask;
  }
  return -1;
}

template <int D>
__device__ __forceinline__ void edge_of(const int32_t* sig, int k, int32_t (&e)[D]) {
#pragma unroll
  for (int a = 0, b = 0; a <= D; ++a)
    if (a != k) e[b++] = sig[a];
}

template <int D>
__device__ void bump_edges(const Tables& t, const int32_t (&sig)[D + 1]) {
#pragma unroll 1
  for (int k = 0; k <= D; ++k) {
    int32_t e[D];
    edge_of<D>(sig, k, e);
    bool ins;
    // the inserting bump writes count = 1 before the slot is published (one
    // plain store in the sector being written anyway); only a later bump of a
    // published slot pays the atomic -- about half of all bumps
    const int64_t h = table_insert<D>(t.ekeys, t.estate, t.ecap, e, ins, t.overflow,
                                      [&](int64_t hh) { t.ecount[(int64_t)t.es * hh] = 1; }, t.es);
    if (h >= 0 && !ins) atomicAdd(&t.ecount[(int64_t)t.es * h], 1);
  }
}

template <int D>
__global__ void k_insert_vertices(Tables t, const int32_t* __restrict__ sigma, int64_t nv,
                                  int32_t base_id, int32_t level, int bump) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int32_t s[D + 1];
#pragma unroll
  for (int a = 0; a <= D; ++a) s[a] = sigma[v * (D + 1) + a];
  bool ins;
  table_insert<D + 1>(t.vkeys, t.vstate, t.vcap, s, ins, t.overflow, [&](int64_t h) {
    t.vval[h] = base_id + (int32_t)v;
    t.vlevel[h] = level;
  });
  if (bump) bump_edges<D>(t, s);
}

// Re-insert the published edge slots of an old edge table (grow / rehash).
template <int D>
__global__ void k_rehash_edges(Tables t, const int32_t* __restrict__ okeys,
                               const int32_t* __restrict__ ostate,
                               const int32_t* __restrict__ ocount, int64_t ocap) {
  const int64_t h0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int os = edge_stride_dev(ostate, ocount);
  if (h0 >= ocap || ostate[(int64_t)os * h0] != 2) return;
  int32_t e[D];
#pragma unroll
  for (int a = 0; a < D; ++a) e[a] = okeys[h0 * D + a];
  const int32_t c = ocount[(int64_t)os * h0];
  bool ins;
  table_insert<D>(t.ekeys, t.estate, t.ecap, e, ins, t.overflow,
                  [&](int64_t h) { t.ecount[(int64_t)t.es * h] = c; }, t.es);
}

// (sub_n, sub_j): sub-rounds of a level -- only the frontier vertices with
// v % sub_n == sub_j open their edges in this round (the others report none).
template <int D>
__device__ __forceinline__ void open_edges_one(Tables t, const int32_t* sigma, int64_t nv,
                             uint8_t* open_mask, int32_t* open_count, int64_t v,
                             int sub_n = 1, int sub_j = 0) {
  if (v >= nv) return;
  if (sub_n > 1 && (int)(v % sub_n) != sub_j) {
#pragma unroll
    for (int k = 0; k <= D; ++k) open_mask[v * (D + 1) + k] = 0;
    open_count[v] = 0;
    return;
  }
  const int32_t* s = sigma + v * (D + 1);
  int cnt = 0;
#pragma unroll 1
  for (int k = 0; k <= D; ++k) {
    int32_t e[D];
    edge_of<D>(s, k, e);
    const int64_t h = table_find<D>(t.ekeys, t.estate, t.ecap, e, t.es);
    const int c = h >= 0 ? __ldcg(t.ecount + (int64_t)t.es * h) : 0;
    const bool open = c < 2;
    open_mask[v * (D + 1) + k] = open ? 1 : 0;
    cnt += open;
  }
  open_count[v] = cnt;
}

template <int D>
__global__ void k_open_edges(Tables t, const int32_t* __restrict__ sigma, int64_t nv,
                             uint8_t* __restrict__ open_mask, int32_t* __restrict__ open_count,
                             int sub_n, int sub_j) {
  open_edges_one<D>(t, sigma, nv, open_mask, open_count,
                    blockIdx.x * (int64_t)blockDim.x + threadIdx.x, sub_n, sub_j);
}

// One thread per frontier vertex: LU of D (rows x_s - x_s0) once, then the
// direction of every open edge (raycast.py:363-377).
template <int D>
__device__ __forceinline__ void emit_rays_one(const double* rec, const int32_t* sigma,
                            const double* r, int64_t nv,
                            const uint8_t* open_mask,
                            const int64_t* open_off, double* ray_x, double* ray_u,
                            int32_t* ray_eta, int32_t* ray_parent, int32_t* bad, int64_t v) {
  if (v >= nv) return;
  constexpr int S = rec_stride(D);
  const int32_t* s = sigma + v * (D + 1);
  int64_t o = open_off[v];
  bool any = false;
#pragma unroll
  for (int k = 0; k <= D; ++k) any |= open_mask[v * (D + 1) + k] != 0;
  if (!any) return;
  const double* x0 = rec + (int64_t)s[0] * S;
  double A[D][D];
  int piv[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double* xa = rec + (int64_t)s[a + 1] * S;
#pragma unroll
    for (int j = 0; j < D; ++j) A[a][j] = xa[j] - x0[j];
  }
  const bool ok = lu_factor<D>(A, piv);
  for (int k = 0; k <= D; ++k) {
    if (!open_mask[v * (D + 1) + k]) continue;
    double w[D];
#pragma unroll
    for (int j = 0; j < D; ++j) w[j] = (k == 0) ? 1.0 : (j == k - 1 ? 1.0 : 0.0);
    if (ok) lu_solve<D>(A, piv, w);
    double nn = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) nn = fma(w[j], w[j], nn);
    const double nrm = sqrt(nn);
    if (!ok || !(nrm > 0.0) || !isfinite(nrm)) atomicAdd(bad, 1);
    const double sc = (k == 0 ? 1.0 : -1.0) / nrm;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      ray_x[o * D + j] = r[v * D + j];
      ray_u[o * D + j] = w[j] * sc;
    }
    int32_t e[D];
    edge_of<D>(s, k, e);
#pragma unroll
    for (int j = 0; j < D; ++j) ray_eta[o * D + j] = e[j];
    ray_parent[o] = (int32_t)v;
    ++o;
  }
}

template <int D>
__global__ void k_emit_rays(const double* __restrict__ rec, const int32_t* __restrict__ sigma,
                            const double* __restrict__ r, int64_t nv,
                            const uint8_t* __restrict__ open_mask,
                            const int64_t* __restrict__ open_off, double* ray_x, double* ray_u,
                            int32_t* ray_eta, int32_t* ray_parent, int32_t* bad) {
  emit_rays_one<D>(rec, sigma, r, nv, open_mask, open_off, ray_x, ray_u, ray_eta, ray_parent, bad, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
}

// sigma' = sorted(eta + {i}); claim the key for the smallest ray id.
template <int D>
__device__ __forceinline__ void claim_one(Tables t, const int32_t* ray_eta,
                        const int32_t* hit_idx, const uint8_t* hit_flag,
                        int64_t n, int32_t level, int32_t* out_sigma,
                        int64_t* out_slot, int64_t k) {
  if (k >= n) return;
  out_slot[k] = -1;
  if (hit_flag[k] != VR_RAY_OK) return;
  const int32_t i = hit_idx[k];
  int32_t s[D + 1];
  int b = 0;
  bool placed = false;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int32_t e = ray_eta[k * D + a];
    if (!placed && i < e) { s[b++] = i; placed = true; }
    s[b++] = e;
  }
  if (!placed) s[b++] = i;
#pragma unroll
  for (int a = 0; a <= D; ++a) out_sigma[k * (D + 1) + a] = s[a];
  bool ins;
  const int64_t h = table_insert<D + 1>(t.vkeys, t.vstate, t.vcap, s, ins, t.overflow,
                                        [&](int64_t hh) {
                                          t.vval[hh] = (int32_t)k;
                                          t.vlevel[hh] = level;
                                        });
  if (h < 0) return;
  if (!ins && __ldcg(t.vlevel + h) == level) atomicMin(&t.vval[h], (int32_t)k);
  out_slot[k] = h;
}

template <int D>
__global__ void k_claim(Tables t, const int32_t* __restrict__ ray_eta,
                        const int32_t* __restrict__ hit_idx, const uint8_t* __restrict__ hit_flag,
                        int64_t n, int32_t level, int32_t* __restrict__ out_sigma,
                        int64_t* __restrict__ out_slot) {
  claim_one<D>(t, ray_eta, hit_idx, hit_flag, n, level, out_sigma, out_slot, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
}

// Claim received sigma rows (owner-sharded traversal): as k_claim with the
// candidate already formed; row k claims with id k (smallest row wins).
template <int D>
__global__ void k_claim_sigma(Tables t, const int32_t* __restrict__ rows, int64_t n,
                              int32_t level, int64_t* __restrict__ out_slot) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t s[D + 1];
#pragma unroll
  for (int a = 0; a <= D; ++a) s[a] = rows[k * (D + 1) + a];
  bool ins;
  const int64_t h = table_insert<D + 1>(t.vkeys, t.vstate, t.vcap, s, ins, t.overflow,
                                        [&](int64_t hh) {
                                          t.vval[hh] = (int32_t)k;
                                          t.vlevel[hh] = level;
                                        });
  if (h >= 0 && !ins && __ldcg(t.vlevel + h) == level) atomicMin(&t.vval[h], (int32_t)k);
  out_slot[k] = h;
}

__global__ void k_winners_sigma(Tables t, const int64_t* __restrict__ slot, int64_t n,
                                int32_t level, int32_t* __restrict__ new_flag) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t h = slot[k];
  new_flag[k] = (h >= 0 && t.vlevel[h] == level && t.vval[h] == (int32_t)k) ? 1 : 0;
}

// Edge-owner side of the sharded bump: +1 per received key (insert-or-find),
// then, after every bump of the level, the count of each key.
template <int D>
__global__ void k_bump_keys(Tables t, const int32_t* __restrict__ keys, int64_t n) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t e[D];
#pragma unroll
  for (int a = 0; a < D; ++a) e[a] = keys[k * D + a];
  bool ins;
  const int64_t h = table_insert<D>(t.ekeys, t.estate, t.ecap, e, ins, t.overflow,
                                    [&](int64_t hh) { t.ecount[(int64_t)t.es * hh] = 1; }, t.es);
  if (h >= 0 && !ins) atomicAdd(&t.ecount[(int64_t)t.es * h], 1);
}

template <int D>
__global__ void k_edge_counts(Tables t, const int32_t* __restrict__ keys, int64_t n,
                              int32_t* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t e[D];
#pragma unroll
  for (int a = 0; a < D; ++a) e[a] = keys[k * D + a];
  const int64_t h = table_find<D>(t.ekeys, t.estate, t.ecap, e, t.es);
  out[k] = h >= 0 ? __ldcg(t.ecount + (int64_t)t.es * h) : 0;
}

template <int D>
__device__ __forceinline__ void winners_one(Tables t, const int64_t* slot,
                          const uint8_t* hit_flag, int64_t n, int32_t level,
                          int32_t* new_flag, int32_t* esc_flag, int64_t k) {
  if (k >= n) return;
  const int64_t h = slot[k];
  new_flag[k] = (h >= 0 && t.vlevel[h] == level && t.vval[h] == (int32_t)k) ? 1 : 0;
  esc_flag[k] = hit_flag[k] == VR_RAY_ESCAPED ? 1 : 0;
}

template <int D>
__global__ void k_winners(Tables t, const int64_t* __restrict__ slot,
                          const uint8_t* __restrict__ hit_flag, int64_t n, int32_t level,
                          int32_t* __restrict__ new_flag, int32_t* __restrict__ esc_flag) {
  winners_one<D>(t, slot, hit_flag, n, level, new_flag, esc_flag, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
}

template <int D>
__device__ __forceinline__ void finalize_one(Tables t, const double* rec,
                           const int32_t* ray_sigma,
                           const int64_t* slot, const int32_t* new_flag,
                           const int64_t* new_off, int64_t n, int32_t base_id,
                           int32_t* vsig, double* vr,
                           int32_t* bad, int64_t k) {
  if (k >= n || !new_flag[k]) return;
  constexpr int S = rec_stride(D);
  const int64_t id = base_id + new_off[k];
  int32_t s[D + 1];
#pragma unroll
  for (int a = 0; a <= D; ++a) {
    s[a] = ray_sigma[k * (D + 1) + a];
    vsig[id * (D + 1) + a] = s[a];
  }
  // fresh fp64 circumcentre (centred at x_s0) -- no chained drift
  const double* x0 = rec + (int64_t)s[0] * S;
  double A[D][D], b[D];
  int piv[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double* xa = rec + (int64_t)s[a + 1] * S;
    double q = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double e = xa[j] - x0[j];
      A[a][j] = 2.0 * e;
      q = fma(e, e, q);
    }
    b[a] = q;
  }
  const bool ok = lu_factor<D>(A, piv);
  if (ok) lu_solve<D>(A, piv, b);
  else atomicAdd(bad, 1);
#pragma unroll
  for (int j = 0; j < D; ++j) vr[id * D + j] = x0[j] + b[j];
  t.vval[slot[k]] = (int32_t)id;
}

template <int D>
__global__ void k_finalize(Tables t, const double* __restrict__ rec,
                           const int32_t* __restrict__ ray_sigma,
                           const int64_t* __restrict__ slot, const int32_t* __restrict__ new_flag,
                           const int64_t* __restrict__ new_off, int64_t n, int32_t base_id,
                           int32_t* __restrict__ vsig, double* __restrict__ vr,
                           int32_t* __restrict__ bad) {
  finalize_one<D>(t, rec, ray_sigma, slot, new_flag, new_off, n, base_id, vsig, vr, bad, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
}

// The d+1 edge-count bumps of every new vertex (graph.py:115-120), split from
// k_finalize: the hash probes are latency-bound and want full occupancy,
// while the fp64 circumcentre solve holds ~200 registers (10 warps/SM; config
// 5: the fused kernel took 116 ms of the traversal's GPU time).
template <int D>
__device__ __forceinline__ void bump_new_one(Tables t, const int32_t* ray_sigma,
                           const int32_t* new_flag, int64_t n, int64_t k) {
  if (k >= n || !new_flag[k]) return;
  int32_t s[D + 1];
#pragma unroll
  for (int a = 0; a <= D; ++a) s[a] = ray_sigma[k * (D + 1) + a];
  bump_edges<D>(t, s);
}

template <int D>
__global__ void k_bump_new(Tables t, const int32_t* __restrict__ ray_sigma,
                           const int32_t* __restrict__ new_flag, int64_t n) {
  bump_new_one<D>(t, ray_sigma, new_flag, n, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
}

template <int D>
__device__ __forceinline__ void boundary_one(const int32_t* esc_flag,
                           const int64_t* esc_off,
                           const int32_t* ray_parent,
                           const double* ray_u, int64_t n,
                           const int32_t* frontier_sigma, int64_t base_b,
                           int32_t* bsig, double* bu, int64_t k) {
  if (k >= n || !esc_flag[k]) return;
  const int64_t b = base_b + esc_off[k];
  const int32_t p = ray_parent[k];
#pragma unroll
  for (int a = 0; a <= D; ++a) bsig[b * (D + 1) + a] = frontier_sigma[(int64_t)p * (D + 1) + a];
#pragma unroll
  for (int j = 0; j < D; ++j) bu[b * D + j] = ray_u[k * D + j];
}

template <int D>
__global__ void k_boundary(const int32_t* __restrict__ esc_flag,
                           const int64_t* __restrict__ esc_off,
                           const int32_t* __restrict__ ray_parent,
                           const double* __restrict__ ray_u, int64_t n,
                           const int32_t* __restrict__ frontier_sigma, int64_t base_b,
                           int32_t* __restrict__ bsig, double* __restrict__ bu) {
  boundary_one<D>(esc_flag, esc_off, ray_parent, ray_u, n, frontier_sigma, base_b, bsig, bu, blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
}

template <int D>
__global__ void k_edge_compact(Tables t, const int64_t* __restrict__ off,
                               int32_t* __restrict__ out_keys, int32_t* __restrict__ out_count) {
  const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (h >= t.ecap || t.estate[(int64_t)t.es * h] != 2) return;
  const int64_t o = off[h];
#pragma unroll
  for (int a = 0; a < D; ++a) out_keys[o * D + a] = t.ekeys[h * D + a];
  out_count[o] = t.ecount[(int64_t)t.es * h];
}

__global__ void k_published(const int32_t* __restrict__ state, int64_t cap, int32_t* flag) {
  const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (h < cap) flag[h] = state[h] == 2 ? 1 : 0;
}

}  // namespace
