// Monte-Carlo cell volumes and interface areas:
// Philox directions -> fused RayCast -> per-cell segmented reduction in ray
// order (reference integrate_mc.py:124-197).
#include "raycast_core.cuh"

using namespace vr;

namespace {

constexpr int RED_NT = 256;
constexpr int RED_CHUNK = 1024;   // rays per reduction chunk (4 per thread)
constexpr int RED_MAPCAP = 1024;  // minimum face map capacity (max_faces <= 512)
// Face maps larger than this many bytes live in a caller workspace in global
// memory instead of dynamic shared memory (unbounded face counts).
constexpr int RED_SMEM_MAP_MAX = 160 * 1024;

__host__ __device__ constexpr int map_entry_bytes(bool integ) { return integ ? 24 : 16; }

inline int map_capacity(int max_faces) {
  int cap = RED_MAPCAP;
  while (cap < 2 * max_faces) cap *= 2;
  return cap;
}

// Integrand on the device for the CLI's built-ins (reference integrands.py):
// kind 1 const c, 2 sin(x_1^2), 3 linear a.x + b.
struct Integ {
  int kind;      // 0: areas/volume only
  int m;         // subsamples per ray
  double coef[VR_MAX_D_ALL + 1];
  const double* unif;  // nullable: replayed uniforms (n_rays, m); else Philox
};

template <int D>
__device__ __forceinline__ double integrand(const Integ& f, const double (&p)[D]) {
  if (f.kind == 1) return f.coef[0];
  if (f.kind == 2) return sin(p[0] * p[0]);
  double v = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) v = fma(f.coef[k], p[k], v);
  return v + f.coef[D];
}

// Subsample uniform s of ray `ray` of generator `cell`: Philox counter
// (ray, cell, 0x100 + s/2, 'MU'), two 53-bit uniforms in [0, 1) per call.
__device__ __forceinline__ double philox_uniform(uint64_t seed, int64_t cell, int64_t ray, int s) {
  uint32_t c[4] = {(uint32_t)ray, (uint32_t)cell,
                   (0x100u + (uint32_t)(s >> 1)) | ((uint32_t)(ray >> 32) << 16),
                   0x4D550000u | (uint32_t)((cell >> 32) & 0xFFFF)};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t a = (s & 1) ? ((((uint64_t)c[2]) << 32) | c[3]) : ((((uint64_t)c[0]) << 32) | c[1]);
  return (double)(a >> 11) * 0x1.0p-53;
}

template <int D, bool INTEG>
__global__ void __launch_bounds__(RED_NT)
    k_mc_reduce(SrcMC<D> src, const int32_t* __restrict__ ray_idx, const double* __restrict__ ray_t,
                const uint8_t* __restrict__ ray_flag, int max_faces, int degenerate_is_error,
                double surf, Integ fi, double* out_volume, int32_t* out_face_j,
                double* out_face_area, int32_t* out_nfaces, int32_t* out_status,
                int64_t* out_first_bad, double* out_samples, double* out_face_surf,
                double* out_vol_integral, const int32_t* __restrict__ cell_sel, int mapcap,
                unsigned char* __restrict__ gmap) {
  constexpr int S = rec_stride(D);
  constexpr int CH = INTEG ? 512 : RED_CHUNK;  // rays per chunk (smem budget)
  __shared__ unsigned long long keys[CH];  // (face << 32 | ray) per ray of the chunk, ~0 if none
  __shared__ double wv[CH];
  __shared__ double lv[CH];
  __shared__ double sv[INTEG ? CH : 1];   // f(rp) w          (integrate_mc.py:350)
  __shared__ double fv[INTEG ? CH : 1];   // acc * length^d   (integrate_mc.py:356)
  __shared__ int rslot[CH];          // face-map slot of each ray of the chunk (-1: none)
  __shared__ unsigned long long first_bad;  // (ray << 2) | kind
  __shared__ int nused;  // faces (+ mapcap per face that found no slot: OVERFLOW)
  __shared__ int nface;  // entries of flist
  // face map (mapcap entries): accumulators, keys (neighbour index, -1 free)
  // and the slots in insertion order -- in dynamic shared memory, or in the
  // caller's global workspace for very large face counts
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  unsigned char* mbase =
      gmap ? gmap + (size_t)blockIdx.x * mapcap * map_entry_bytes(INTEG) : dyn_smem;
  double* macc = reinterpret_cast<double*>(mbase);
  double* macc2 = macc + mapcap;  // INTEG only
  int* mkey = reinterpret_cast<int*>(macc + (INTEG ? 2 : 1) * (size_t)mapcap);
  int* flist = mkey + mapcap;

  // block b reduces cell row cell_sel[b] (all rows without a selection);
  // its outputs go to row b
  const int64_t o = blockIdx.x;
  const int64_t c = cell_sel ? (int64_t)cell_sel[o] : o;
  const int64_t per = src.per;
  const int32_t cell = src.cells[c];
  const double* xc = src.grec + (int64_t)cell * S;
  for (int i = threadIdx.x; i < mapcap; i += RED_NT) {
    mkey[i] = -1;
    macc[i] = 0.0;
    if (INTEG) macc2[i] = 0.0;
  }
  if (threadIdx.x == 0) { first_bad = ~0ull; nused = 0; nface = 0; }
  double vol = 0.0, fvol = 0.0;  // lane 0 of the last warp: sequential sums in ray order
  __syncthreads();

  for (int64_t start = 0; start < per; start += CH) {
    const int cnt = (int)min((int64_t)CH, per - start);
    for (int s = threadIdx.x; s < CH; s += RED_NT) {
      unsigned long long key = ~0ull;
      double w = 0.0, ld = 0.0, sw = 0.0, fl_v = 0.0;
      if (s < cnt) {
        const int64_t r = start + s;
        const int64_t k = c * per + r;
        const uint8_t fl = ray_flag[k];
        const bool bad = fl == VR_RAY_ESCAPED || (fl == VR_RAY_DEGENERATE && degenerate_is_error);
        if (bad) {
          atomicMin(&first_bad, ((unsigned long long)r << 2) | (fl == VR_RAY_ESCAPED ? 1ull : 2ull));
          if (out_samples) out_samples[k] = CUDART_NAN;
        } else {
          const int32_t j = ray_idx[k];
          const double t = ray_t[k];
          double y[D], rp[D], seg[D];
          src.direction(k, y);
          const double* xj = src.grec + (int64_t)j * S;
          double ss = 0.0, nd = 0.0, nn = 0.0;
#pragma unroll
          for (int q = 0; q < D; ++q) {
            rp[q] = fma(t, y[q], xc[q]);  // rp = xi + t y  (raycast.py:210)
            seg[q] = rp[q] - xc[q];       // integrate_mc.py:151
            ss = fma(seg[q], seg[q], ss);
            const double nij = xj[q] - xc[q];
            nd = fma(nij, y[q], nd);
            nn = fma(nij, nij, nn);
          }
          const double length = sqrt(ss);
          const double cosang = nd / sqrt(nn);
          double p = 1.0;
#pragma unroll
          for (int q = 0; q < D - 1; ++q) p *= length;
          w = p / cosang;          // length^(d-1) / cos
          ld = p * length;         // length^d
          key = ((unsigned long long)(uint32_t)j << 32) | (unsigned)s;
          if (out_samples) out_samples[k] = ld;
          if constexpr (INTEG) {
            sw = integrand<D>(fi, rp) * w;
            double acc = 0.0;
            for (int m = 0; m < fi.m; ++m) {
              const double tm = fi.unif ? fi.unif[k * fi.m + m]
                                        : philox_uniform(src.seed, cell, r, m);
              double pt[D];
#pragma unroll
              for (int q = 0; q < D; ++q) pt[q] = fma(tm, seg[q], xc[q]);
              double tp = 1.0;
#pragma unroll
              for (int q = 0; q < D - 1; ++q) tp *= tm;
              acc += integrand<D>(fi, pt) * tp;  // integrate_mc.py:354-355
            }
            fl_v = acc * ld;
          }
        }
      }
      keys[s] = key;
      wv[s] = w;
      lv[s] = ld;
      if constexpr (INTEG) {
        sv[s] = sw;
        fv[s] = fl_v;
      }
    }
    __syncthreads();
    // Each ray's face slot (insert-or-find in the face map; a new face is
    // appended to flist).
    for (int s = threadIdx.x; s < cnt; s += RED_NT) {
      const unsigned long long key = keys[s];
      int slot = -1;
      if (key != ~0ull) {
        const uint32_t j = (uint32_t)(key >> 32);
        unsigned h = (j * 2654435761u) & (mapcap - 1);
        for (int probe = 0; probe < mapcap; ++probe) {
          const int prev = atomicCAS(&mkey[h], -1, (int)j);
          if (prev == -1) {
            atomicAdd(&nused, 1);
            flist[atomicAdd(&nface, 1)] = (int)h;
            slot = (int)h;
            break;
          }
          if (prev == (int)j) { slot = (int)h; break; }
          h = (h + 1) & (mapcap - 1);
        }
        if (slot < 0) atomicAdd(&nused, mapcap);  // map full: reported as OVERFLOW
      }
      rslot[s] = slot;
    }
    __syncthreads();
    constexpr int NWR = RED_NT / 32;
    if (threadIdx.x == RED_NT - 32) {  // volume: sequential sum in ray order (integrate_mc.py:156),
      for (int s = 0; s < cnt; ++s) {  // on the last warp, which takes no faces
        vol += lv[s];
        if (INTEG) fvol += fv[s];
      }
    }
    // Per face, the weights of its rays summed in ray order (the reference's
    // accumulation order): one warp per face finds the face's rays 32 at a
    // time with a ballot, lane 0 adds them in order.  (Replaces a bitonic
    // sort of the (face, ray) keys: 55 block-wide stages per chunk.)
    {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      const int nf_now = nface;
      for (int f = warp; warp < NWR - 1 && f < nf_now; f += NWR - 1) {
        const int slot = flist[f];
        // continue the face's running sums: one sequential sum in ray order
        // across chunks (integrate_mc.py:154-155)
        double sum = macc[slot], sum2 = INTEG ? macc2[slot] : 0.0;
        for (int base = 0; base < cnt; base += 32) {
          const int s = base + lane;
          unsigned m = __ballot_sync(0xffffffffu, s < cnt && rslot[s] == slot);
          if (lane == 0) {
            while (m) {
              const int q = base + __ffs(m) - 1;
              m &= m - 1;
              sum += wv[q];
              if (INTEG) sum2 += sv[q];
            }
          }
        }
        if (lane == 0) {
          macc[slot] = sum;  // one writer per face per chunk
          if (INTEG) macc2[slot] = sum2;
        }
      }
    }
    __syncthreads();
  }

  // Emit faces sorted by neighbour index: a face's position is the number of
  // faces with a smaller index (distinct indices).
  const int nf = nused;
  const int nl = nface;
  const double scale = surf / (double)per;  // integrate_mc.py:357-358
  for (int f = threadIdx.x; f < nl; f += RED_NT) {
    const int slot = flist[f];
    const int j = mkey[slot];
    int p = 0;
    for (int g = 0; g < nl; ++g) p += mkey[flist[g]] < j ? 1 : 0;
    if (p < max_faces) {
      out_face_j[o * max_faces + p] = j;
      out_face_area[o * max_faces + p] = macc[slot] * scale;
      if (INTEG) out_face_surf[o * max_faces + p] = macc2[slot] * scale;
    }
  }
  if (threadIdx.x == RED_NT - 32) {
    out_volume[o] = vol * surf / (double)((int64_t)D * per);  // integrate_mc.py:359-360
    if (INTEG) out_vol_integral[o] = fvol * surf / (double)(per * (int64_t)fi.m);  // :363
    out_nfaces[o] = nf < max_faces ? nf : max_faces;
    int status = VR_CELL_OK;
    int64_t fb = -1;
    if (first_bad != ~0ull) {
      fb = (int64_t)(first_bad >> 2);
      status = (first_bad & 3ull) == 1ull ? VR_CELL_UNBOUNDED : VR_CELL_DEGENERATE;
    } else if (nf > max_faces) {
      status = VR_CELL_OVERFLOW;
    }
    out_status[o] = status;
    out_first_bad[o] = fb;
  }
}

template <int D>
__global__ void k_mc_dirs(SrcMC<D> src, double* out_z) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= src.n) return;
  const int64_t c = k / src.per;
  double z[D];
  philox_normals<D>(src.seed, src.cells[c], k - c * src.per, z);
#pragma unroll
  for (int j = 0; j < D; ++j) out_z[k * D + j] = z[j];
}

}  // namespace

extern "C" int vr_mc_rays(const double* rec, int64_t n_gen, int d, double sqmax,
                          const vr_screen32* s32, const double* cand_rec, const int32_t* cand, int64_t n_cand,
                          const int32_t* cells, int64_t n_cells, int64_t rays_per_cell,
                          const double* dirs, uint64_t seed, int32_t* out_idx, double* out_t,
                          uint8_t* out_flag, int32_t* recheck_list, int32_t* recheck_count,
                          void* stream) {
  if (!rec || !cells || !out_idx || !out_t || !out_flag || rays_per_cell <= 0) return VR_EINVAL;
  const double* crec = cand ? cand_rec : rec;
  const int64_t nc = cand ? n_cand : n_gen;
  if (!crec || nc <= 0) return VR_EINVAL;
  const int64_t n = n_cells * rays_per_cell;
  RayOut out{out_idx, out_t, nullptr, out_flag, recheck_list, recheck_count};
  if (d > VR_MAX_D) {
    if (s32) return VR_EDIM;  // fp32 screen: d <= 8
    VR_DISPATCH_D_HIGH(d, {
      SrcMC<D> src{rec, cells, rays_per_cell, dirs, seed, n};
      return launch_raycast_fp64<D>(src, n, crec, cand, nc, make_screen(sqmax, nullptr, d), out,
                                    as_stream(stream));
    });
  }
  VR_DISPATCH_D(d, {
    SrcMC<D> src{rec, cells, rays_per_cell, dirs, seed, n};
    return launch_raycast<D>(src, n, crec, cand, nc, make_screen(sqmax, s32, d), out,
                             as_stream(stream));
  });
  return VR_OK;
}

extern "C" int vr_mc_recheck(const double* rec, int64_t n_gen, int d, const double* cand_rec,
                             const int32_t* cand, int64_t n_cand, const int32_t* cells,
                             int64_t rays_per_cell, const double* dirs, uint64_t seed,
                             const int32_t* recheck_list, const int32_t* recheck_count,
                             int64_t max_list, int32_t* out_idx, double* out_t, uint8_t* out_flag,
                             void* stream) {
  if (!rec || !cells || !recheck_list || !recheck_count) return VR_EINVAL;
  const double* crec = cand ? cand_rec : rec;
  const int64_t nc = cand ? n_cand : n_gen;
  RayOut out{out_idx, out_t, nullptr, out_flag, nullptr, nullptr};
  VR_DISPATCH_D_ALL(d, {
    SrcMC<D> src{rec, cells, rays_per_cell, dirs, seed, INT64_MAX};
    return launch_recheck<D>(src, max_list, crec, cand, nc, recheck_list, recheck_count, out,
                             as_stream(stream));
  });
  return VR_OK;
}

namespace {

// Launch k_mc_reduce over n_blocks cell rows (cell_sel: row per block, or
// all rows) with a face map of map_capacity(max_faces) entries, in dynamic
// shared memory up to RED_SMEM_MAP_MAX bytes, else in map_ws.
template <int D, bool INTEG>
int launch_reduce(const SrcMC<D>& src, int64_t n_blocks, const int32_t* ray_idx,
                  const double* ray_t, const uint8_t* ray_flag, int max_faces,
                  int degenerate_is_error, double surf, const Integ& fi, double* out_volume,
                  int32_t* out_face_j, double* out_face_area, int32_t* out_nfaces,
                  int32_t* out_status, int64_t* out_first_bad, double* out_samples,
                  double* out_face_surf, double* out_vol_integral, const int32_t* cell_sel,
                  void* map_ws, int64_t map_ws_bytes, cudaStream_t st) {
  const int cap = map_capacity(max_faces);
  const int64_t map_bytes = (int64_t)cap * map_entry_bytes(INTEG);
  unsigned char* gmap = nullptr;
  int smem = 0;
  if (map_bytes > RED_SMEM_MAP_MAX) {
    if (!map_ws || map_ws_bytes < map_bytes * n_blocks) return VR_ECAPACITY;
    gmap = static_cast<unsigned char*>(map_ws);
  } else {
    smem = (int)map_bytes;
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
      cudaError_t e = cudaFuncSetAttribute(k_mc_reduce<D, INTEG>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           RED_SMEM_MAP_MAX);
      if (e != cudaSuccess) return vr_cuda_status(e);
      attr_set = true;
    }
  }
  k_mc_reduce<D, INTEG><<<(unsigned)n_blocks, RED_NT, smem, st>>>(
      src, ray_idx, ray_t, ray_flag, max_faces, degenerate_is_error, surf, fi, out_volume,
      out_face_j, out_face_area, out_nfaces, out_status, out_first_bad, out_samples,
      out_face_surf, out_vol_integral, cell_sel, cap, gmap);
  VR_RETURN_LAUNCH();
}

}  // namespace

extern "C" int64_t vr_mc_map_bytes(int64_t n_blocks, int max_faces, int integrate) {
  if (n_blocks <= 0 || max_faces <= 0) return 0;
  const int64_t map_bytes = (int64_t)map_capacity(max_faces) * map_entry_bytes(integrate != 0);
  return map_bytes > RED_SMEM_MAP_MAX ? map_bytes * n_blocks : 0;
}

extern "C" int vr_mc_reduce(const double* rec, int d, const int32_t* cells, int64_t n_cells,
                            int64_t rays_per_cell, const double* dirs, uint64_t seed,
                            const int32_t* ray_idx, const double* ray_t, const uint8_t* ray_flag,
                            int max_faces, int degenerate_is_error, double surf,
                            const int32_t* cell_sel, int64_t n_sel, void* map_ws,
                            int64_t map_ws_bytes, double* out_volume, int32_t* out_face_j,
                            double* out_face_area, int32_t* out_nfaces, int32_t* out_status,
                            int64_t* out_first_bad, double* out_samples, void* stream) {
  if (!rec || !cells || !ray_idx || !ray_t || !ray_flag || !out_volume || !out_face_j ||
      !out_face_area || !out_nfaces || !out_status || !out_first_bad)
    return VR_EINVAL;
  if (max_faces <= 0 || max_faces > (1 << 28)) return VR_EINVAL;
  const int64_t nb = cell_sel ? n_sel : n_cells;
  if (nb <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    SrcMC<D> src{rec, cells, rays_per_cell, dirs, seed, n_cells * rays_per_cell};
    Integ fi{};
    return launch_reduce<D, false>(src, nb, ray_idx, ray_t, ray_flag, max_faces,
                                   degenerate_is_error, surf, fi, out_volume, out_face_j,
                                   out_face_area, out_nfaces, out_status, out_first_bad,
                                   out_samples, nullptr, nullptr, cell_sel, map_ws, map_ws_bytes,
                                   as_stream(stream));
  });
  return VR_OK;
}

extern "C" int vr_mc_integrate(const double* rec, int d, const int32_t* cells, int64_t n_cells,
                               int64_t rays_per_cell, const double* dirs, uint64_t seed,
                               const int32_t* ray_idx, const double* ray_t,
                               const uint8_t* ray_flag, int max_faces, double surf,
                               int integrand_kind, const double* coef, int m_sub,
                               const double* unif, const int32_t* cell_sel, int64_t n_sel,
                               void* map_ws, int64_t map_ws_bytes, double* out_volume,
                               int32_t* out_face_j, double* out_face_area, double* out_face_surf,
                               double* out_vol_integral, int32_t* out_nfaces,
                               int32_t* out_status, int64_t* out_first_bad, void* stream) {
  if (!rec || !cells || !ray_idx || !ray_t || !ray_flag || !out_volume || !out_face_j ||
      !out_face_area || !out_face_surf || !out_vol_integral || !out_nfaces || !out_status ||
      !out_first_bad || m_sub < 1 || integrand_kind < 1 || integrand_kind > 3)
    return VR_EINVAL;
  if (max_faces <= 0 || max_faces > (1 << 28)) return VR_EINVAL;
  const int64_t nb = cell_sel ? n_sel : n_cells;
  if (nb <= 0) return VR_OK;
  Integ fi{};
  fi.kind = integrand_kind;
  fi.m = m_sub;
  fi.unif = unif;
  const int ncoef = integrand_kind == 1 ? 1 : (integrand_kind == 3 ? d + 1 : 0);
  for (int k = 0; k < ncoef; ++k) fi.coef[k] = coef[k];
  VR_DISPATCH_D_ALL(d, {
    SrcMC<D> src{rec, cells, rays_per_cell, dirs, seed, n_cells * rays_per_cell};
    return launch_reduce<D, true>(src, nb, ray_idx, ray_t, ray_flag, max_faces, 1, surf, fi,
                                  out_volume, out_face_j, out_face_area, out_nfaces, out_status,
                                  out_first_bad, nullptr, out_face_surf, out_vol_integral,
                                  cell_sel, map_ws, map_ws_bytes, as_stream(stream));
  });
  return VR_OK;
}

extern "C" int vr_mc_uniforms(int64_t n_cells, const int32_t* cells, int64_t rays_per_cell,
                              int m_sub, uint64_t seed, double* out_u, void* stream);

extern "C" int vr_mc_directions(int d, int64_t n_cells, const int32_t* cells,
                                int64_t rays_per_cell, uint64_t seed, double* out_z,
                                void* stream) {
  if (!cells || !out_z || rays_per_cell <= 0) return VR_EINVAL;
  const int64_t n = n_cells * rays_per_cell;
  if (n <= 0) return VR_OK;
  VR_DISPATCH_D_ALL(d, {
    SrcMC<D> src{nullptr, cells, rays_per_cell, nullptr, seed, n};
    k_mc_dirs<D><<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(src, out_z);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_mc_rays_pruned(const double* rec, int64_t n_gen, int d, double sqmax,
                                 const vr_screen32* s32, const vr_prune_index* ix, const int32_t* cells, int64_t n_cells,
                                 int64_t rays_per_cell, const double* dirs, uint64_t seed,
                                 const int32_t* order, int32_t* out_idx, double* out_t,
                                 uint8_t* out_flag, int32_t* recheck_list,
                                 int32_t* recheck_count, uint64_t* work,
                                 void* stream) {
  if (!rec || !ix || !ix->rec || !cells || !out_idx || !out_t || !out_flag || rays_per_cell <= 0 ||
      ix->n != n_gen)
    return VR_EINVAL;
  const int64_t n = n_cells * rays_per_cell;
  RayOut out{out_idx, out_t, nullptr, out_flag, recheck_list, recheck_count};
  const PrunedIndex pi = pruned_index_from(ix, s32 != nullptr);
  const Screen sc = make_screen(sqmax, s32, d);
  VR_DISPATCH_D(d, {
    SrcMC<D> src{rec, cells, rays_per_cell, dirs, seed, n};
    src.order = order;
    return launch_raycast_pruned<D>(src, n, pi, sc.fr, out, as_stream(stream),
                                    reinterpret_cast<unsigned long long*>(work));
  });
  return VR_OK;
}

namespace {
__global__ void k_mc_unif(const int32_t* cells, int64_t per, int64_t n, int m, uint64_t seed,
                          double* out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t c = k / per;
  for (int s = 0; s < m; ++s) out[k * m + s] = philox_uniform(seed, cells[c], k - c * per, s);
}
}  // namespace

extern "C" int vr_mc_uniforms(int64_t n_cells, const int32_t* cells, int64_t rays_per_cell,
                              int m_sub, uint64_t seed, double* out_u, void* stream) {
  if (!cells || !out_u || rays_per_cell <= 0 || m_sub < 1) return VR_EINVAL;
  const int64_t n = n_cells * rays_per_cell;
  if (n <= 0) return VR_OK;
  k_mc_unif<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(cells, rays_per_cell, n,
                                                                        m_sub, seed, out_u);
  VR_RETURN_LAUNCH();
}
