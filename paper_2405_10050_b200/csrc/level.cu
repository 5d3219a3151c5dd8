// Native driver of one level-synchronous traversal level (graph.py:88-146
// restated as a frontier loop).
//
// The per-level work is ~15 kernels plus two host synchronisations (the ray
// count, then the new-vertex / escape counts that size the next level and the
// table growth).  Driving it from Python cost ~0.45 ms of host time per level
// (torch ops, ctypes, stream lookups) -- more than the device work of the
// small levels of configs 1 and 3.  These two entry points run the same
// kernels in the same order from C++ (cub scans and radix sort), so a level
// costs two ctypes calls and two synchronisations:
//
//   vr_trav_level_open:  open edges of the frontier -> exclusive scan -> R
//   vr_trav_level_cast:  edge rays -> processing order -> pruned RayCast +
//                        exact re-check -> claim / winners -> scans -> counts
//
// The caller (DeviceTraversal.level) then grows the edge table if needed and
// calls vr_trav_finalize / vr_trav_boundary as before.  Results are those of
// the Python-driven level (the processing order is the same stable sort).
#include <atomic>
#include <cub/device/device_scan.cuh>

#include <cstdlib>

#include "common.cuh"

extern "C" {
int vr_trav_open_edges_sub(const vr_traverse_tables* tab, int d, const int32_t* sigma,
                           int64_t n_v, int sub_n, int sub_j, uint8_t* open_mask,
                           int32_t* open_count, void* stream);
int vr_trav_open_edges(const vr_traverse_tables* tab, int d, const int32_t* sigma, int64_t n_v,
                       uint8_t* open_mask, int32_t* open_count, void* stream);
int vr_trav_emit_rays(const double* rec, int d, const int32_t* sigma, const double* r,
                      int64_t n_v, const uint8_t* open_mask, const int64_t* open_off,
                      double* ray_x, double* ray_u, int32_t* ray_eta, int32_t* ray_parent,
                      int32_t* bad, void* stream);
int vr_trav_claim(const vr_traverse_tables* tab, int d, const int32_t* ray_eta,
                  const int32_t* hit_idx, const uint8_t* hit_flag, int64_t n_rays,
                  int32_t level, int32_t* out_sigma, int64_t* out_slot, int32_t* new_flag,
                  int32_t* esc_flag, void* stream);
int vr_ray_order(const int32_t* inv_perm, const int32_t* eta, int eta_len,
                 int64_t rays_per_cell, const double* u, int64_t n, int d, int64_t n_base,
                 int32_t* order, void* workspace, int64_t* workspace_bytes, void* stream);
int vr_raycast_pruned(const double* rec, int64_t n_gen, int d, double sqmax,
                      const vr_screen32* s32, const vr_prune_index* ix, const double* x,
                      const double* u, const int32_t* eta, int eta_len, int64_t n_rays,
                      const int32_t* order, int32_t* out_idx, double* out_t, double* out_rp,
                      uint8_t* out_flag, int32_t* recheck_list, int32_t* recheck_count,
                      uint64_t* work, void* stream);
int vr_raycast_recheck(const double* rec, int64_t n_gen, int d, const double* cand_rec,
                       const int32_t* cand, int64_t n_cand, const double* x, const double* u,
                       const int32_t* eta, int eta_len, const int32_t* recheck_list,
                       const int32_t* recheck_count, int64_t max_list, int32_t* out_idx,
                       double* out_t, double* out_rp, uint8_t* out_flag, void* stream);
}

// defaults measured on config 5 (N = 1e6, d = 8, 36.5 M vertices): 2 rounds for
// levels of >= 8 M estimated rays cast 45.9 M instead of 56.6 M edges, 0.787 vs
// 0.826 s; 4 / 8 rounds cast 42.1 / 40.4 M but their sparser batches screen
// more pairs per ray (0.803 / 0.847 s)
#ifndef VR_SUB_RAYS_DEFAULT
#define VR_SUB_RAYS_DEFAULT 4000000
#endif
#ifndef VR_SUB_MAX_DEFAULT
#define VR_SUB_MAX_DEFAULT 2
#endif

namespace {

inline unsigned nbk(int64_t n, int nt = 256) {
  const int64_t b = (n + nt - 1) / nt;
  return (unsigned)(b < 65535 * 16 ? b : 65535 * 16);
}

template <typename T>
__global__ void k_widen(const T* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i];
}

__global__ void k_count_degenerate(const uint8_t* __restrict__ flag, int64_t n,
                                   unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c += flag[i] == 3 ? 1 : 0;
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// cnt[0] += escaped rays, cnt[1] += degenerate rays
__global__ void k_count_flags(const uint8_t* __restrict__ flag, int64_t n,
                              unsigned long long* __restrict__ cnt) {
  unsigned long long esc = 0, deg = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    esc += flag[i] == 1 ? 1 : 0;
    deg += flag[i] == 3 ? 1 : 0;
  }
  for (int off = 16; off > 0; off >>= 1) {
    esc += __shfl_xor_sync(0xffffffffu, esc, off);
    deg += __shfl_xor_sync(0xffffffffu, deg, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (esc) atomicAdd(cnt, esc);
    if (deg) atomicAdd(cnt + 1, deg);
  }
}

__global__ void k_rays_counts(const unsigned long long* __restrict__ cnt,
                              const int32_t* __restrict__ bad, int64_t* __restrict__ counts) {
  counts[0] = (int64_t)cnt[0];
  counts[1] = (int64_t)cnt[1];
  counts[2] = bad[0];
}

// counts[0..4] = n_new, n_esc, n_degenerate, bad frontier vertices, overflow
__global__ void k_level_counts(const int32_t* __restrict__ new_flag,
                               const int64_t* __restrict__ new_off,
                               const int32_t* __restrict__ esc_flag,
                               const int64_t* __restrict__ esc_off, int64_t n,
                               const unsigned long long* __restrict__ ndeg,
                               const int32_t* __restrict__ bad,
                               const int32_t* __restrict__ overflow, int64_t* __restrict__ counts) {
  counts[0] = new_off[n - 1] + new_flag[n - 1];
  counts[1] = esc_off[n - 1] + esc_flag[n - 1];
  counts[2] = (int64_t)*ndeg;
  counts[3] = bad[0];
  counts[4] = overflow[0];
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t scan_tmp_bytes(int64_t n) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int)(n > 0 ? n : 1));
  return tmp;
}

// Exclusive int64 scan of an int32 array (cub) with caller scratch.
cudaError_t excl_scan(const int32_t* in, int64_t* out, int64_t n, void* tmp, size_t tmp_bytes,
                      cudaStream_t st) {
  // widen into `out`, then scan in place (cub allows in == out for scans)
  k_widen<int32_t><<<nbk(n), 256, 0, st>>>(in, out, n);
  return cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, out, out, (int)n, st);
}

// Scratch layout of vr_trav_level_cast (R rays): order, recheck list / count,
// degenerate counter, device counts, then scratch shared by the ray-order
// sort and the scans.
struct CastPlan {
  size_t o_order, o_rl, o_rc, o_deg, o_cnt, o_tmp, tmp, total;
};

int cast_plan(int64_t R, int64_t n_gen, int d, CastPlan& p) {
  int64_t order_ws = 0;
  int s = vr_ray_order(nullptr, nullptr, d, 1, nullptr, R, d, n_gen, nullptr, nullptr, &order_ws,
                       nullptr);
  if (s) return s;
  const size_t scan = scan_tmp_bytes(R);
  p.tmp = (size_t)order_ws > scan ? (size_t)order_ws : scan;
  p.o_order = 0;
  p.o_rl = align256(p.o_order + 4 * R);
  p.o_rc = align256(p.o_rl + 4 * R);
  p.o_deg = align256(p.o_rc + 4);
  p.o_cnt = align256(p.o_deg + 16);
  p.o_tmp = align256(p.o_cnt + 8 * 5);
  p.total = p.o_tmp + p.tmp;
  return VR_OK;
}

int fail(cudaError_t e) { return e == cudaSuccess ? VR_OK : vr_cuda_status(e); }

}  // namespace

extern "C" int vr_trav_level_workspace(int64_t n_v, int64_t n_rays, int64_t n_gen, int d,
                                       int64_t* bytes) {
  if (!bytes || n_v < 0 || n_rays < 0) return VR_EINVAL;
  size_t need = align256(scan_tmp_bytes(n_v));
  if (n_rays > 0) {
    CastPlan p;
    int s = cast_plan(n_rays, n_gen, d, p);
    if (s) return s;
    if (p.total > need) need = p.total;
  }
  *bytes = (int64_t)need;
  return VR_OK;
}

namespace {
int level_open_sub(const vr_traverse_tables* tab, int d, const int32_t* frontier_sigma,
                   int64_t n_v, int sub_n, int sub_j, uint8_t* open_mask, int32_t* open_count,
                   int64_t* open_off, int64_t* n_rays_out, void* workspace,
                   int64_t workspace_bytes, void* stream);
}

extern "C" int vr_trav_level_open(const vr_traverse_tables* tab, int d,
                                  const int32_t* frontier_sigma, int64_t n_v, uint8_t* open_mask,
                                  int32_t* open_count, int64_t* open_off, int64_t* n_rays_out,
                                  void* workspace, int64_t workspace_bytes, void* stream) {
  return level_open_sub(tab, d, frontier_sigma, n_v, 1, 0, open_mask, open_count, open_off,
                        n_rays_out, workspace, workspace_bytes, stream);
}

namespace {
int level_open_sub(const vr_traverse_tables* tab, int d, const int32_t* frontier_sigma,
                   int64_t n_v, int sub_n, int sub_j, uint8_t* open_mask, int32_t* open_count,
                   int64_t* open_off, int64_t* n_rays_out, void* workspace,
                   int64_t workspace_bytes, void* stream) {
  if (!tab || !frontier_sigma || !open_mask || !open_count || !open_off || !n_rays_out)
    return VR_EINVAL;
  *n_rays_out = 0;
  if (n_v <= 0) return VR_OK;
  if (n_v >= (int64_t)1 << 31) return VR_EINVAL;  // cub scans with int counts
  const size_t tmp = scan_tmp_bytes(n_v);
  if (!workspace || workspace_bytes < (int64_t)tmp) return VR_ECAPACITY;
  cudaStream_t st = as_stream(stream);
  int s = vr_trav_open_edges_sub(tab, d, frontier_sigma, n_v, sub_n, sub_j, open_mask, open_count,
                                 stream);
  if (s) return s;
  cudaError_t e = excl_scan(open_count, open_off, n_v, workspace, tmp, st);
  if (e != cudaSuccess) return fail(e);
  int64_t last[1];
  int32_t cnt[1];
  if ((e = cudaMemcpyAsync(last, open_off + n_v - 1, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(cnt, open_count + n_v - 1, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return fail(e);
  *n_rays_out = last[0] + cnt[0];
  return VR_OK;
}
}  // namespace

extern "C" int vr_trav_level_cast(
    const vr_traverse_tables* tab, const double* rec, int64_t n_gen, int d, double sqmax,
    const vr_screen32* s32, const vr_prune_index* ix, const int32_t* frontier_sigma,
    const double* frontier_r, int64_t n_v, const uint8_t* open_mask, const int64_t* open_off,
    int64_t n_rays, int32_t level, double* ray_x, double* ray_u, int32_t* ray_eta,
    int32_t* ray_parent, int32_t* hit_idx, double* hit_t, uint8_t* hit_flag, int32_t* ray_sigma,
    int64_t* slot, int32_t* new_flag, int32_t* esc_flag, int64_t* new_off, int64_t* esc_off,
    int32_t* bad, uint64_t* work, int64_t* counts_out, void* workspace, int64_t workspace_bytes,
    void* stream) {
  if (!tab || !rec || !ix || !ix->inv_perm || !frontier_sigma || !frontier_r || !open_mask ||
      !open_off || !ray_x || !ray_u || !ray_eta || !ray_parent || !hit_idx || !hit_t ||
      !hit_flag || !ray_sigma || !slot || !new_flag || !esc_flag || !new_off || !esc_off ||
      !bad || !counts_out)
    return VR_EINVAL;
  for (int i = 0; i < 5; ++i) counts_out[i] = 0;
  if (n_rays <= 0) return VR_OK;
  if (n_rays >= (int64_t)1 << 31) return VR_EINVAL;
  const int64_t R = n_rays;
  CastPlan P;
  int s = cast_plan(R, n_gen, d, P);
  if (s) return s;
  if (!workspace || workspace_bytes < (int64_t)P.total) return VR_ECAPACITY;
  cudaStream_t st = as_stream(stream);
  cudaError_t e;
  if ((e = cudaMemsetAsync(bad, 0, 2 * sizeof(int32_t), st)) != cudaSuccess) return fail(e);
  s = vr_trav_emit_rays(rec, d, frontier_sigma, frontier_r, n_v, open_mask, open_off, ray_x,
                        ray_u, ray_eta, ray_parent, bad, stream);
  if (s) return s;
  char* base = static_cast<char*>(workspace);
  int32_t* order = reinterpret_cast<int32_t*>(base + P.o_order);
  int32_t* rl = reinterpret_cast<int32_t*>(base + P.o_rl);
  int32_t* rc = reinterpret_cast<int32_t*>(base + P.o_rc);
  unsigned long long* ndeg = reinterpret_cast<unsigned long long*>(base + P.o_deg);
  int64_t* dcounts = reinterpret_cast<int64_t*>(base + P.o_cnt);
  void* tmp = base + P.o_tmp;
  // processing order (raycast.py coherent_order: stable sort of the keys)
  int64_t tb = (int64_t)P.tmp;
  s = vr_ray_order(ix->inv_perm, ray_eta, d, 1, ray_u, R, d, n_gen, order, tmp, &tb, stream);
  if (s) return s;
  // RayCast of the level's edge rays (|eta| = d) + exact re-check
  s = vr_raycast_pruned(rec, n_gen, d, sqmax, s32, ix, ray_x, ray_u, ray_eta, d, R, order,
                        hit_idx, hit_t, nullptr, hit_flag, rl, rc, work, stream);
  if (s) return s;
  s = vr_raycast_recheck(rec, n_gen, d, nullptr, nullptr, 0, ray_x, ray_u, ray_eta, d, rl, rc, R,
                         hit_idx, hit_t, nullptr, hit_flag, stream);
  if (s) return s;
  // claim the hit vertices, then offsets of the new vertices / escapes
  s = vr_trav_claim(tab, d, ray_eta, hit_idx, hit_flag, R, level, ray_sigma, slot, new_flag,
                    esc_flag, stream);
  if (s) return s;
  if ((e = excl_scan(new_flag, new_off, R, tmp, P.tmp, st)) != cudaSuccess) return fail(e);
  if ((e = excl_scan(esc_flag, esc_off, R, tmp, P.tmp, st)) != cudaSuccess) return fail(e);
  if ((e = cudaMemsetAsync(ndeg, 0, 8, st)) != cudaSuccess) return fail(e);
  k_count_degenerate<<<nbk(R, 256) < 1184 ? nbk(R, 256) : 1184, 256, 0, st>>>(hit_flag, R, ndeg);
  k_level_counts<<<1, 1, 0, st>>>(new_flag, new_off, esc_flag, esc_off, R, ndeg, bad,
                                  tab->overflow, dcounts);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpyAsync(counts_out, dcounts, 5 * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return fail(e);
  return VR_OK;
}

// The rays of one level without the local claim (owner-sharded traversal:
// the hits go to their owners).  counts_out[3] = {escapes, degenerate rays,
// affinely dependent frontier vertices}.
extern "C" int vr_trav_level_rays(const double* rec, int64_t n_gen, int d, double sqmax,
                                  const vr_screen32* s32, const vr_prune_index* ix,
                                  const int32_t* frontier_sigma, const double* frontier_r,
                                  int64_t n_v, const uint8_t* open_mask, const int64_t* open_off,
                                  int64_t n_rays, double* ray_x, double* ray_u, int32_t* ray_eta,
                                  int32_t* ray_parent, int32_t* hit_idx, double* hit_t,
                                  uint8_t* hit_flag, int32_t* bad, uint64_t* work,
                                  int64_t* counts_out, void* workspace, int64_t workspace_bytes,
                                  void* stream) {
  if (!rec || !ix || !ix->inv_perm || !frontier_sigma || !frontier_r || !open_mask ||
      !open_off || !ray_x || !ray_u || !ray_eta || !ray_parent || !hit_idx || !hit_t ||
      !hit_flag || !bad || !counts_out)
    return VR_EINVAL;
  for (int i = 0; i < 3; ++i) counts_out[i] = 0;
  if (n_rays <= 0) return VR_OK;
  if (n_rays >= (int64_t)1 << 31) return VR_EINVAL;
  const int64_t R = n_rays;
  CastPlan P;
  int s = cast_plan(R, n_gen, d, P);
  if (s) return s;
  if (!workspace || workspace_bytes < (int64_t)P.total) return VR_ECAPACITY;
  cudaStream_t st = as_stream(stream);
  cudaError_t e;
  if ((e = cudaMemsetAsync(bad, 0, 2 * sizeof(int32_t), st)) != cudaSuccess) return fail(e);
  s = vr_trav_emit_rays(rec, d, frontier_sigma, frontier_r, n_v, open_mask, open_off, ray_x,
                        ray_u, ray_eta, ray_parent, bad, stream);
  if (s) return s;
  char* base = static_cast<char*>(workspace);
  int32_t* order = reinterpret_cast<int32_t*>(base + P.o_order);
  int32_t* rl = reinterpret_cast<int32_t*>(base + P.o_rl);
  int32_t* rc = reinterpret_cast<int32_t*>(base + P.o_rc);
  unsigned long long* ndeg = reinterpret_cast<unsigned long long*>(base + P.o_deg);
  int64_t* dcounts = reinterpret_cast<int64_t*>(base + P.o_cnt);
  void* tmp = base + P.o_tmp;
  int64_t tb = (int64_t)P.tmp;
  s = vr_ray_order(ix->inv_perm, ray_eta, d, 1, ray_u, R, d, n_gen, order, tmp, &tb, stream);
  if (s) return s;
  s = vr_raycast_pruned(rec, n_gen, d, sqmax, s32, ix, ray_x, ray_u, ray_eta, d, R, order,
                        hit_idx, hit_t, nullptr, hit_flag, rl, rc, work, stream);
  if (s) return s;
  s = vr_raycast_recheck(rec, n_gen, d, nullptr, nullptr, 0, ray_x, ray_u, ray_eta, d, rl, rc, R,
                         hit_idx, hit_t, nullptr, hit_flag, stream);
  if (s) return s;
  if ((e = cudaMemsetAsync(ndeg, 0, 16, st)) != cudaSuccess) return fail(e);
  const unsigned g = nbk(R, 256) < 1184 ? nbk(R, 256) : 1184;
  k_count_flags<<<g, 256, 0, st>>>(hit_flag, R, ndeg);
  k_rays_counts<<<1, 1, 0, st>>>(ndeg, bad, dcounts);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpyAsync(counts_out, dcounts, 3 * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return fail(e);
  return VR_OK;
}

// ---------------------------------------------------------------------------
// Native multi-level driver (vr_trav_run): the level loop itself in C++.
// Each level is open -> (capacity checks) -> cast -> finalize + boundary,
// with the two host synchronisations of the level calls and nothing else on
// the host; it returns to the caller only when the traversal is done, the
// level limit is reached, or a capacity (workspace, vertex arrays / table,
// edge table, boundary arrays) must grow -- the caller grows it and calls
// again (state->phase records whether the current level's cast is done).
// ---------------------------------------------------------------------------
extern "C" {
int vr_trav_finalize(const vr_traverse_tables* tab, const double* rec, int d,
                     const int32_t* ray_sigma, const int64_t* slot, const int32_t* new_flag,
                     const int64_t* new_off, int64_t n_rays, int32_t base_id, int32_t* vsig,
                     double* vr, int32_t* bad, int bump, void* stream);
int vr_trav_boundary(int d, const int32_t* esc_flag, const int64_t* esc_off,
                     const int32_t* ray_parent, const double* ray_u, int64_t n_rays,
                     const int32_t* frontier_sigma, int64_t base_b, int32_t* bsig, double* bu,
                     void* stream);
}

namespace vr {
int trav_run_small(const vr_traverse_tables* tab, vr_trav_state* S, const double* rec,
                   int64_t n_gen, int d, double sqmax, const vr_screen32* s32,
                   const vr_prune_index* ix, int32_t last_level, int64_t* level_new,
                   int64_t level_cap, uint64_t* work, void* workspace, int64_t workspace_bytes,
                   cudaStream_t st, int* handled, int32_t* bail_code);
int64_t small_rmax(int d);  // rays per level the persistent kernel takes
}

namespace {

// Sub-rounds of a large level.  A level-synchronous traversal casts one ray
// per open edge of the frontier, so a new vertex adjacent to k frontier
// vertices is found k times (config 5: 56.6 M rays for 36.5 M vertices); the
// reference's one-vertex-at-a-time loop (graph.py:122-145) casts it once,
// because the first discovery closes the other k - 1 edges (graph.py:115-120).
// Splitting the frontier into sub_n interleaved sub-rounds (vertex v of the
// frontier belongs to round v % sub_n; each round opens, casts, claims,
// stores and bumps before the next one opens) recovers part of that: a ray
// is skipped whenever an earlier round already found its far vertex.  The
// vertex set, edge counts and boundary rays are those of the unsplit level.
// A level of F frontier vertices is split so that a round casts about
// VR_SUB_RAYS rays (estimated as F (d + 1) / 2), at most VR_SUB_MAX rounds.
std::atomic<int64_t> g_sub_rays{-1};  // vr_trav_set_sub_rounds overrides (-1: environment / default)
std::atomic<int> g_sub_max{-1};
int64_t sub_target_rays() {
  const int64_t o = g_sub_rays.load(std::memory_order_relaxed);
  if (o >= 0) return o;
  static const int64_t v = [] {
    const char* e = std::getenv("VR_SUB_RAYS");
    return e ? (int64_t)std::atoll(e) : (int64_t)VR_SUB_RAYS_DEFAULT;
  }();
  return v;
}
int sub_max_rounds() {
  int m = g_sub_max.load(std::memory_order_relaxed);
  if (m < 0) {
    static const int v = [] {
      const char* e = std::getenv("VR_SUB_MAX");
      return e ? std::atoi(e) : VR_SUB_MAX_DEFAULT;
    }();
    m = v;
  }
  return m < 1 ? 1 : (m > 64 ? 64 : m);
}
int plan_sub_rounds(int64_t F, int d) {
  const int64_t target = sub_target_rays();
  if (target <= 0) return 1;
  const int64_t est = F * (d + 1) / 2;
  int64_t n = est / target;
  if (n < 1) n = 1;
  if (n > sub_max_rounds()) n = sub_max_rounds();
  return (int)n;
}
// claim epoch of (level, sub-round): distinct from every level number the
// other paths tag their claims with
int32_t claim_epoch(int32_t level, int sub_j) { return 0x40000000 + level * 64 + sub_j; }

// VR_SMALL_LEVELS=0 disables the persistent small-level kernel (A/B runs).
bool small_mode() {
  const char* e = std::getenv("VR_SMALL_LEVELS");
  return !e || std::atoi(e) != 0;
}

// Per-level buffers carved from the caller's workspace (F frontier
// vertices, R rays), then the scratch of the two level calls.
struct RunPlan {
  size_t o_mask, o_cnt, o_off, o_x, o_u, o_eta, o_par, o_hidx, o_ht, o_hflag, o_rsig, o_slot,
      o_newf, o_escf, o_noff, o_eoff, o_bad, o_scr, scratch, total;
};

int run_plan(int64_t F, int64_t R, int64_t n_gen, int d, RunPlan& p) {
  int64_t scr = 0;
  int s = vr_trav_level_workspace(F, R, n_gen, d, &scr);
  if (s) return s;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align256(o + bytes);
    return at;
  };
  p.o_mask = take((size_t)F * (d + 1));
  p.o_cnt = take(4 * (size_t)F);
  p.o_off = take(8 * (size_t)F);
  p.o_x = take(8 * (size_t)R * d);
  p.o_u = take(8 * (size_t)R * d);
  p.o_eta = take(4 * (size_t)R * d);
  p.o_par = take(4 * (size_t)R);
  p.o_hidx = take(4 * (size_t)R);
  p.o_ht = take(8 * (size_t)R);
  p.o_hflag = take((size_t)R);
  p.o_rsig = take(4 * (size_t)R * (d + 1));
  p.o_slot = take(8 * (size_t)R);
  p.o_newf = take(4 * (size_t)R);
  p.o_escf = take(4 * (size_t)R);
  p.o_noff = take(8 * (size_t)R);
  p.o_eoff = take(8 * (size_t)R);
  p.o_bad = take(16);
  p.scratch = (size_t)scr;
  p.o_scr = take(p.scratch);
  p.total = o;
  return VR_OK;
}

}  // namespace

extern "C" int vr_trav_set_sub_rounds(int64_t rays_per_round, int max_rounds) {
  g_sub_rays.store(rays_per_round, std::memory_order_relaxed);
  g_sub_max.store(max_rounds, std::memory_order_relaxed);
  return VR_OK;
}

extern "C" int vr_trav_run_workspace(int64_t n_frontier, int64_t n_rays, int64_t n_gen, int d,
                                     int64_t* bytes) {
  if (!bytes) return VR_EINVAL;
  RunPlan p;
  const int s = run_plan(n_frontier, n_rays, n_gen, d, p);
  if (s) return s;
  *bytes = (int64_t)p.total;
  return VR_OK;
}

extern "C" int vr_trav_run(const vr_traverse_tables* tab, vr_trav_state* S, const double* rec,
                           int64_t n_gen, int d, double sqmax, const vr_screen32* s32,
                           const vr_prune_index* ix, int32_t last_level, int64_t* level_new,
                           int64_t level_cap, uint64_t* work, void* workspace,
                           int64_t workspace_bytes, void* stream) {
  if (!tab || !S || !rec || !ix || !level_new) return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  char* W = static_cast<char*>(workspace);
  S->need = VR_RUN_DONE;
  int32_t host_level = -1;  // a level the persistent kernel handed back
  while (true) {
    const int64_t F = S->f1 - S->f0;
    if (F <= 0 || (last_level >= 0 && S->level > last_level)) {
      S->need = VR_RUN_DONE;
      return VR_OK;
    }
    if (S->level >= level_cap) return VR_ECAPACITY;
    // small levels: the persistent kernel (level_small.cu) runs as many as
    // stay small in one launch
    // (expected rays ~ F (d+1) / 2: about half the edges of a frontier
    // vertex are open; larger levels skip the attempt)
    if (S->phase == 0 && S->sub_j == 0 && S->level != host_level && small_mode() &&
        F * (d + 1) <= 2 * vr::small_rmax(d)) {
      int handled = 0;
      int32_t bail = 0;
      const int s0 = vr::trav_run_small(tab, S, rec, n_gen, d, sqmax, s32, ix, last_level,
                                        level_new, level_cap, work, workspace, workspace_bytes,
                                        st, &handled, &bail);
      if (s0) return s0;
      if (handled) {
        if (S->need != bail) return VR_OK;  // done, error, or a capacity to grow
        host_level = S->level;               // this level is too large: host path
        S->need = VR_RUN_DONE;
        continue;
      }
    }
    const int32_t* fs = S->vsig + S->f0 * (d + 1);
    const double* fr = S->vr + S->f0 * d;
    // workspace for the open step (R unknown yet: R <= (d+1) F)
    RunPlan p0;
    int s = run_plan(F, 0, n_gen, d, p0);
    if (s) return s;
    if (!workspace || workspace_bytes < (int64_t)p0.total) {
      S->need = VR_RUN_NEED_WORKSPACE;
      S->need_amount = (int64_t)p0.total;
      return VR_OK;
    }
    uint8_t* mask = reinterpret_cast<uint8_t*>(W + p0.o_mask);
    int32_t* ocnt = reinterpret_cast<int32_t*>(W + p0.o_cnt);
    int64_t* ooff = reinterpret_cast<int64_t*>(W + p0.o_off);
    int64_t R = S->pending_rays;
    if (S->phase == 0) {
      if (S->sub_j == 0) {  // the level starts: its vertices go to ids f1 ..
        S->nv = S->f1;
        S->sub_n = plan_sub_rounds(F, d);
      }
      s = level_open_sub(tab, d, fs, F, S->sub_n, S->sub_j, mask, ocnt, ooff, &R, W + p0.o_scr,
                         (int64_t)p0.scratch, stream);
      if (s) return s;
      if (R == 0) {  // nothing open in this round
        if (++S->sub_j < S->sub_n) continue;
        S->sub_j = 0;
        const bool grew = S->nv > S->f1;
        S->f0 = S->f1;
        S->f1 = S->nv;
        S->level += 1;
        if (grew) continue;
        S->need = VR_RUN_DONE;  // nothing open in the whole level: the traversal ends here
        return VR_OK;
      }
      S->pending_rays = R;
      // the open result (mask, counts, offsets: the workspace prefix) stays
      // valid across capacity returns: growing the tables does not change an
      // edge count, and the caller keeps the prefix when the workspace grows
      // (re-opening the last config-5 level cost ~17 ms per return)
      S->phase = 2;
    }
    RunPlan p;
    if ((s = run_plan(F, R, n_gen, d, p))) return s;
    if (workspace_bytes < (int64_t)p.total) {
      S->need = VR_RUN_NEED_WORKSPACE;
      S->need_amount = (int64_t)p.total;
      return VR_OK;
    }
    // the open step's buffers sit at the same offsets in both plans
    double* rx = reinterpret_cast<double*>(W + p.o_x);
    double* ru = reinterpret_cast<double*>(W + p.o_u);
    int32_t* reta = reinterpret_cast<int32_t*>(W + p.o_eta);
    int32_t* rpar = reinterpret_cast<int32_t*>(W + p.o_par);
    int32_t* hidx = reinterpret_cast<int32_t*>(W + p.o_hidx);
    double* ht = reinterpret_cast<double*>(W + p.o_ht);
    uint8_t* hflag = reinterpret_cast<uint8_t*>(W + p.o_hflag);
    int32_t* rsig = reinterpret_cast<int32_t*>(W + p.o_rsig);
    int64_t* slot = reinterpret_cast<int64_t*>(W + p.o_slot);
    int32_t* newf = reinterpret_cast<int32_t*>(W + p.o_newf);
    int32_t* escf = reinterpret_cast<int32_t*>(W + p.o_escf);
    int64_t* noff = reinterpret_cast<int64_t*>(W + p.o_noff);
    int64_t* eoff = reinterpret_cast<int64_t*>(W + p.o_eoff);
    int32_t* bad = reinterpret_cast<int32_t*>(W + p.o_bad);
    if (S->phase == 2) {
      // capacity for up to R new vertices (arrays; vertex table at load <= 0.5)
      // and their edges (edge table at load <= 0.5 of the incidence count)
      if (S->nv + R > S->vcap_arrays || 2 * (S->nv + R) > tab->vcap) {
        S->need = VR_RUN_NEED_VERTICES;
        S->need_amount = S->nv + R;
        return VR_OK;
      }
      if (2 * (S->e_ub + (d + 1) * R) > tab->ecap) {
        S->need = VR_RUN_NEED_EDGES;
        S->need_amount = S->e_ub + (d + 1) * R;
        return VR_OK;
      }
      int64_t counts[5];
      s = vr_trav_level_cast(tab, rec, n_gen, d, sqmax, s32, ix, fs, fr, F, mask, ooff, R,
                             claim_epoch(S->level, S->sub_j), rx, ru, reta, rpar, hidx, ht, hflag,
                             rsig, slot, newf,
                             escf, noff, eoff, bad, work, counts, W + p.o_scr,
                             (int64_t)p.scratch, stream);
      if (s) return s;
      S->n_new = counts[0];
      S->n_esc = counts[1];
      S->n_degenerate = counts[2];
      S->n_bad = counts[3];
      S->overflow = counts[4];
      if (S->n_degenerate || S->n_bad || S->overflow) {
        S->need = VR_RUN_ERROR;
        return VR_OK;
      }
      S->phase = 1;
    }
    // phase 1: the cast is done -- store the new vertices, bump their edges,
    // record the boundary rays
    if (S->nb + S->n_esc > S->bcap) {
      S->need = VR_RUN_NEED_BOUNDARY;
      S->need_amount = S->nb + S->n_esc;
      return VR_OK;
    }
    s = vr_trav_finalize(tab, rec, d, rsig, slot, newf, noff, R, (int32_t)S->nv, S->vsig, S->vr,
                         bad + 1, 1, stream);
    if (s) return s;
    if (S->n_esc) {
      s = vr_trav_boundary(d, escf, eoff, rpar, ru, R, fs, S->nb, S->bsig, S->bu, stream);
      if (s) return s;
    }
    S->e_ub += (d + 1) * S->n_new;
    S->nb += S->n_esc;
    S->nv += S->n_new;
    level_new[S->level] += S->n_new;
    S->rays += R;
    S->phase = 0;
    S->pending_rays = 0;
    if (++S->sub_j >= S->sub_n) {  // the level is complete
      S->sub_j = 0;
      S->f0 = S->f1;
      S->f1 = S->nv;
      S->level += 1;
    }
  }
}
