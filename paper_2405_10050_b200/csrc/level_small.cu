// Persistent small-level traversal: whole levels of the level-synchronous
// traversal (graph.py:88-146) in ONE cooperative kernel launch, phases
// separated by grid-wide barriers instead of kernel boundaries and host
// synchronisations.
//
// The per-level host path (level.cu) costs ~25 launches and two host syncs
// per level -- ~180 us, whatever the level size.  A small diagram (config 1:
// 32 levels of a few hundred vertices) is all latency: 5.7 ms of 7.1.  Here a
// level is nine grid barriers (~2 us each) around the same per-element
// bodies (trav_core.cuh) and the same cooperative warp-per-ray RayCast
// (coop_ray) the host path uses for batches below 8192 rays, so the mesh is
// bitwise the host path's: same ray order (frontier order, open-edge rank),
// same claim rule (the smallest ray id wins a new sigma), same ids (prefix
// sums over the winners), same fp64 circumcentres.  The kernel keeps going
// while levels stay small (F, R <= 8192); a larger level, a capacity limit,
// an error or the end of the traversal hands control back to vr_trav_run
// through the device copy of vr_trav_state.
#include <cooperative_groups.h>

#include <atomic>

#include "raycast_core.cuh"
#include "trav_core.cuh"

namespace cg = cooperative_groups;
using namespace vr;

namespace {

constexpr int SM_NT = 256;
constexpr int SM_NW = SM_NT / 32;
constexpr int32_t NEED_CONTINUE = -1;
constexpr int32_t NEED_BAIL = 100;  // level too large: the host path runs it

struct SmallBufs {
  uint8_t* open_mask;
  int32_t* open_count;
  int64_t* open_off;
  double* ray_x;
  double* ray_u;
  int32_t* ray_eta;
  int32_t* ray_parent;
  int32_t* hit_idx;
  double* hit_t;
  uint8_t* hit_flag;
  int32_t* ray_sigma;
  int64_t* slot;
  int32_t* new_flag;
  int32_t* esc_flag;
  int64_t* new_off;
  int64_t* esc_off;
  int32_t* rl;     // re-check list
  int32_t* rc;     // re-check count
  int32_t* bad;    // [0] singular frontier simplices, [1] singular circumcentres
  unsigned long long* ndeg;
  vr_trav_state* S;
  int64_t* level_new;
};

// Exclusive scan of in[0, n) by one block (every block runs it: n <= 8192,
// cheaper than a grid barrier); out[i] is written only for the elements this
// block owns in the grid-stride loops of the next phase (i / SM_NT ==
// blockIdx.x mod gridDim.x), so the block reads them back after a
// __syncthreads.  Returns the total.
__device__ int64_t block_scan(const int32_t* in, int64_t* out, int64_t n, int64_t* sh) {
  const int64_t per = (n + SM_NT - 1) / SM_NT;
  const int64_t lo = min(n, (int64_t)threadIdx.x * per), hi = min(n, lo + per);
  int64_t sum = 0;
  for (int64_t i = lo; i < hi; ++i) sum += __ldcg(in + i);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t inc = sum;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += o;
  }
  __syncthreads();
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int k = 0; k < SM_NW; ++k) {
      const int64_t v = sh[k];
      sh[k] = run;
      run += v;
    }
    sh[SM_NW] = run;
  }
  __syncthreads();
  int64_t run = sh[w] + inc - sum;
  for (int64_t i = lo; i < hi; ++i) {
    if ((uint64_t)(i / SM_NT) % gridDim.x == blockIdx.x) out[i] = run;
    run += __ldcg(in + i);
  }
  const int64_t total = sh[SM_NW];
  __syncthreads();
  return total;
}

template <int D>
__global__ void __launch_bounds__(SM_NT)
    k_trav_small(Tables t, const double* rec, int64_t n_gen, PrunedIndex ix, Frame fr,
                 SmallBufs B, int32_t last_level, int64_t level_cap, int64_t fmax, int64_t rmax,
                 unsigned long long* work) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int stk[SM_NW][COOP_STK];
  __shared__ double sh_t[SM_NW];
  __shared__ int sh_i[SM_NW];
  __shared__ int64_t sh_scan[SM_NW + 1];
  volatile vr_trav_state* S = B.S;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t gwarp = gtid >> 5, nwarps = gstride >> 5;
  const bool lead = gtid == 0;
  if (lead) {
    *B.rc = 0;
    B.bad[0] = B.bad[1] = 0;
    *B.ndeg = 0ull;
  }
  grid.sync();
  for (;;) {
    const int64_t f0 = S->f0, f1 = S->f1, F = f1 - f0;
    const int32_t level = S->level;
    if (F <= 0 || (last_level >= 0 && level > last_level)) {
      if (lead) S->need = VR_RUN_DONE;
      return;
    }
    if (F > fmax || level >= level_cap) {
      if (lead) S->need = NEED_BAIL;
      return;
    }
    const int32_t* fs = S->vsig + f0 * (D + 1);
    const double* frr = S->vr + f0 * D;
    // open edges of the frontier (graph.py:127-128)
    for (int64_t v = gtid; v < F; v += gstride) open_edges_one<D>(t, fs, F, B.open_mask, B.open_count, v);
    grid.sync();
    // ray offsets, ray count, capacity checks (as vr_trav_run's); every block
    // decides the same from the same counts
    const int64_t R = block_scan(B.open_count, B.open_off, F, sh_scan);
    {
      int32_t need = NEED_CONTINUE;
      int64_t amount = 0;
      const int64_t nv = S->nv;
      if (R == 0) {
        need = VR_RUN_DONE;
      } else if (R > rmax) {
        need = NEED_BAIL;
      } else if (nv + R > S->vcap_arrays || 2 * (nv + R) > t.vcap) {
        need = VR_RUN_NEED_VERTICES;
        amount = nv + R;
      } else if (2 * (S->e_ub + (D + 1) * R) > t.ecap) {
        need = VR_RUN_NEED_EDGES;
        amount = S->e_ub + (D + 1) * R;
      } else if (S->nb + R > S->bcap) {
        need = VR_RUN_NEED_BOUNDARY;
        amount = S->nb + R;
      }
      if (need != NEED_CONTINUE) {
        if (lead) {
          if (R == 0) {
            B.level_new[level] = 0;
            S->f0 = f1;
            S->level = level + 1;
          }
          S->need_amount = amount;
          S->need = need;
        }
        return;
      }
    }
    // one ray per open edge (raycast.py:345-378)
    for (int64_t v = gtid; v < F; v += gstride)
      emit_rays_one<D>(rec, fs, frr, F, B.open_mask, B.open_off, B.ray_x, B.ray_u, B.ray_eta,
                       B.ray_parent, B.bad, v);
    grid.sync();
    // the RayCast: one warp per ray (the host path's kernel for < 8192 rays)
    const SrcExplicit<D> src{B.ray_x, B.ray_u, B.ray_eta, D, rec, R, nullptr};
    const RayOut out{B.hit_idx, B.hit_t, nullptr, B.hit_flag, B.rl, B.rc};
    for (int64_t k = gwarp; k < R; k += nwarps)
      coop_ray<D, PRUNE_TILE>(src, k, ix.crec, ix.crec32, ix.perm, ix.inv_perm, ix.wide, fr, out,
                              work, stk[threadIdx.x >> 5]);
    grid.sync();
    // exact re-check of the flagged rays (rare), one block per ray
    const int32_t nrc = *(volatile int32_t*)B.rc;
    if (nrc > 0) {
      const RayOut rout{B.hit_idx, B.hit_t, nullptr, B.hit_flag, nullptr, nullptr};
      for (int32_t li = blockIdx.x; li < nrc; li += gridDim.x)
        recheck_ray<D, SM_NT>(src, __ldcg(B.rl + li), rec, nullptr, n_gen, rout, sh_t, sh_i);
      grid.sync();
    }
    // claim sigma' = sorted(eta + {i}) (smallest ray id wins a new key)
    for (int64_t k = gtid; k < R; k += gstride)
      claim_one<D>(t, B.ray_eta, B.hit_idx, B.hit_flag, R, level, B.ray_sigma, B.slot, k);
    grid.sync();
    for (int64_t k = gtid; k < R; k += gstride) {
      winners_one<D>(t, B.slot, B.hit_flag, R, level, B.new_flag, B.esc_flag, k);
      if (__ldcg(B.hit_flag + k) == VR_RAY_DEGENERATE) atomicAdd(B.ndeg, 1ull);
    }
    grid.sync();
    // ids of the new vertices / boundary rays in ray order (every block)
    const int64_t n_new = block_scan(B.new_flag, B.new_off, R, sh_scan);
    const int64_t n_esc = block_scan(B.esc_flag, B.esc_off, R, sh_scan);
    const unsigned long long ndeg = *(volatile unsigned long long*)B.ndeg;
    const int32_t nbad = *(volatile int32_t*)B.bad;
    const int32_t ovf = *(volatile int32_t*)t.overflow;
    if (ndeg || nbad || ovf) {
      if (lead) {
        S->n_new = n_new;
        S->n_esc = n_esc;
        S->n_degenerate = (int64_t)ndeg;
        S->n_bad = nbad;
        S->overflow = ovf;
        S->need = VR_RUN_ERROR;
      }
      return;
    }
    // store the new vertices (fp64 circumcentres), bump their edges, record
    // the boundary rays (graph.py:115-120, 138-139)
    const int64_t nb0 = S->nb;
    for (int64_t k = gtid; k < R; k += gstride) {
      finalize_one<D>(t, rec, B.ray_sigma, B.slot, B.new_flag, B.new_off, R, (int32_t)f1, S->vsig,
                      S->vr, B.bad + 1, k);
      bump_new_one<D>(t, B.ray_sigma, B.new_flag, R, k);
      boundary_one<D>(B.esc_flag, B.esc_off, B.ray_parent, B.ray_u, R, fs, nb0, S->bsig, S->bu, k);
    }
    grid.sync();
    if (lead) {
      S->n_new = n_new;
      S->n_esc = n_esc;
      S->n_degenerate = S->n_bad = S->overflow = 0;
      S->e_ub += (D + 1) * n_new;
      S->nb = nb0 + n_esc;
      S->nv = f1 + n_new;
      B.level_new[level] = n_new;
      S->rays += R;
      S->f0 = f1;
      S->f1 = f1 + n_new;
      S->level = level + 1;
      *B.rc = 0;  // the next level's counters
      B.bad[0] = B.bad[1] = 0;
      *B.ndeg = 0ull;
    }
    grid.sync();
  }
}

size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

struct SmallPlan {
  size_t o[23];
  size_t total;
};

SmallPlan small_plan(int64_t F, int64_t R, int d, int64_t level_cap) {
  const size_t sz[23] = {(size_t)F * (d + 1), 4 * (size_t)F, 8 * (size_t)F,
                         8 * (size_t)R * d, 8 * (size_t)R * d, 4 * (size_t)R * d, 4 * (size_t)R,
                         4 * (size_t)R, 8 * (size_t)R, (size_t)R, 4 * (size_t)R * (d + 1),
                         8 * (size_t)R, 4 * (size_t)R, 4 * (size_t)R, 8 * (size_t)R,
                         8 * (size_t)R, 4 * (size_t)R, 4, 8, 8, 3 * 8, sizeof(vr_trav_state),
                         8 * (size_t)level_cap};
  SmallPlan p{};
  size_t at = 0;
  for (int i = 0; i < 23; ++i) {
    p.o[i] = at;
    at = a256(at + sz[i]);
  }
  p.total = at;
  return p;
}

// Resident CTAs of the cooperative grid on the current device (one per SM,
// two if registers allow), cached per device.
template <int D>
int small_grid() {
  constexpr int MAXDEV = 64;
  static std::atomic<int> grid[MAXDEV];  // 0: not computed yet
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 0;
  if (dev < MAXDEV) {
    const int g = grid[dev].load(std::memory_order_relaxed);
    if (g > 0) return g;
  }
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_trav_small<D>, SM_NT, 0);
  const int g = sms * (per < 2 ? per : 2);
  if (dev < MAXDEV && g > 0) grid[dev].store(g, std::memory_order_relaxed);
  return g;
}

int small_grid_d(int d) {
  switch (d) {
    case 2: return small_grid<2>();
    case 3: return small_grid<3>();
    case 4: return small_grid<4>();
    case 5: return small_grid<5>();
    case 6: return small_grid<6>();
    case 7: return small_grid<7>();
    case 8: return small_grid<8>();
    default: return 0;
  }
}

template <int D>
int launch_small(const Tables& t, const double* rec, int64_t n_gen, const PrunedIndex& pi,
                 const Frame& fr, const SmallBufs& B, int32_t last_level, int64_t level_cap,
                 int64_t fmax, int64_t rmax, unsigned long long* work, cudaStream_t st) {
  auto kern = k_trav_small<D>;
  const int grid = small_grid<D>();
  if (grid <= 0) return VR_EINVAL;
  Tables tt = t;
  const double* r = rec;
  int64_t ng = n_gen;
  PrunedIndex p = pi;
  Frame f = fr;
  SmallBufs b = B;
  int32_t ll = last_level;
  int64_t lc = level_cap, fm = fmax, rm = rmax;
  unsigned long long* w = work;
  void* args[] = {&tt, &r, &ng, &p, &f, &b, &ll, &lc, &fm, &rm, &w};
  return vr_cuda_status(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(SM_NT),
                                                    args, 0, st));
}

}  // namespace

namespace vr {

int64_t small_rmax(int d) { return 2 * (int64_t)small_grid_d(d) * SM_NW; }

// Levels of the traversal in the persistent kernel while they are small;
// returns VR_OK with *handled = 1 when it ran (S updated; S->need tells the
// caller what happened: NEED_BAIL -> run the current level on the host path).
int trav_run_small(const vr_traverse_tables* tab, vr_trav_state* S, const double* rec,
                   int64_t n_gen, int d, double sqmax, const vr_screen32* s32,
                   const vr_prune_index* ix, int32_t last_level, int64_t* level_new,
                   int64_t level_cap, uint64_t* work, void* workspace, int64_t workspace_bytes,
                   cudaStream_t st, int* handled, int32_t* bail_code) {
  *handled = 0;
  *bail_code = NEED_BAIL;
  if (!s32 || !ix->wide_box32 || ix->wide_levels < 2 || d > 8) return VR_OK;
  // The kernel's register footprint (the union of its phases) allows ~8
  // warps per SM, so a level's rays run in ceil(R / warps) rounds of one
  // warp per ray: levels of up to two rounds stay here (config 3's levels of
  // 3-7 rounds ran 5 ms slower in it than on the host path).
  const int64_t RMAX = small_rmax(d), FMAX = RMAX;
  if (RMAX <= 0) return VR_OK;
  const SmallPlan P = small_plan(FMAX, RMAX, d, level_cap);
  if (!workspace || workspace_bytes < (int64_t)P.total) {
    S->need = VR_RUN_NEED_WORKSPACE;
    S->need_amount = (int64_t)P.total;
    *handled = 1;
    return VR_OK;
  }
  char* W = static_cast<char*>(workspace);
  SmallBufs B;
  B.open_mask = reinterpret_cast<uint8_t*>(W + P.o[0]);
  B.open_count = reinterpret_cast<int32_t*>(W + P.o[1]);
  B.open_off = reinterpret_cast<int64_t*>(W + P.o[2]);
  B.ray_x = reinterpret_cast<double*>(W + P.o[3]);
  B.ray_u = reinterpret_cast<double*>(W + P.o[4]);
  B.ray_eta = reinterpret_cast<int32_t*>(W + P.o[5]);
  B.ray_parent = reinterpret_cast<int32_t*>(W + P.o[6]);
  B.hit_idx = reinterpret_cast<int32_t*>(W + P.o[7]);
  B.hit_t = reinterpret_cast<double*>(W + P.o[8]);
  B.hit_flag = reinterpret_cast<uint8_t*>(W + P.o[9]);
  B.ray_sigma = reinterpret_cast<int32_t*>(W + P.o[10]);
  B.slot = reinterpret_cast<int64_t*>(W + P.o[11]);
  B.new_flag = reinterpret_cast<int32_t*>(W + P.o[12]);
  B.esc_flag = reinterpret_cast<int32_t*>(W + P.o[13]);
  B.new_off = reinterpret_cast<int64_t*>(W + P.o[14]);
  B.esc_off = reinterpret_cast<int64_t*>(W + P.o[15]);
  B.rl = reinterpret_cast<int32_t*>(W + P.o[16]);
  B.rc = reinterpret_cast<int32_t*>(W + P.o[17]);
  B.bad = reinterpret_cast<int32_t*>(W + P.o[18]);
  B.ndeg = reinterpret_cast<unsigned long long*>(W + P.o[19]);
  B.S = reinterpret_cast<vr_trav_state*>(W + P.o[21]);
  B.level_new = reinterpret_cast<int64_t*>(W + P.o[22]);
  const int32_t level0 = S->level;
  cudaError_t e = cudaMemcpyAsync(B.S, S, sizeof(vr_trav_state), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return vr_cuda_status(e);
  const Tables t{tab->vkeys, tab->vstate, tab->vval, tab->vlevel, tab->vcap,
                 tab->ekeys, tab->estate, tab->ecount, tab->ecap, tab->overflow,
                 edge_stride(tab->estate, tab->ecount)};
  const PrunedIndex pi = pruned_index_from(ix, true);
  const Screen sc = make_screen(sqmax, s32, d);
  int s = VR_OK;
  unsigned long long* wk = reinterpret_cast<unsigned long long*>(work);
  switch (d) {
    case 2: s = launch_small<2>(t, rec, n_gen, pi, sc.fr, B, last_level, level_cap, FMAX, RMAX, wk, st); break;
    case 3: s = launch_small<3>(t, rec, n_gen, pi, sc.fr, B, last_level, level_cap, FMAX, RMAX, wk, st); break;
    case 4: s = launch_small<4>(t, rec, n_gen, pi, sc.fr, B, last_level, level_cap, FMAX, RMAX, wk, st); break;
    case 5: s = launch_small<5>(t, rec, n_gen, pi, sc.fr, B, last_level, level_cap, FMAX, RMAX, wk, st); break;
    case 6: s = launch_small<6>(t, rec, n_gen, pi, sc.fr, B, last_level, level_cap, FMAX, RMAX, wk, st); break;
    case 7: s = launch_small<7>(t, rec, n_gen, pi, sc.fr, B, last_level, level_cap, FMAX, RMAX, wk, st); break;
    case 8: s = launch_small<8>(t, rec, n_gen, pi, sc.fr, B, last_level, level_cap, FMAX, RMAX, wk, st); break;
    default: return VR_OK;
  }
  if (s) return s;
  if ((e = cudaMemcpyAsync(S, B.S, sizeof(vr_trav_state), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return vr_cuda_status(e);
  const int32_t level1 = S->level;
  if (level1 > level0) {
    if ((e = cudaMemcpy(level_new + level0, B.level_new + level0, 8 * (size_t)(level1 - level0),
                        cudaMemcpyDeviceToHost)) != cudaSuccess)
      return vr_cuda_status(e);
  }
  *handled = 1;
  return VR_OK;
}

}  // namespace vr
