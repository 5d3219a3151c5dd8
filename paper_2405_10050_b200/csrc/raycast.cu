// C-ABI entry points for the batched incircle RayCast (include/voronray_b200.h).
#include "raycast_core.cuh"

#include <cstdlib>

using namespace vr;

int vr::raycast_variant() {
  static int v = [] {
    const char* e = std::getenv("VR_RAYCAST_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// Tensor-core screen of the pruned kernel (d <= 6, index built with recB):
// on unless VR_MMA=0.
int vr::mma_mode() {
  static int v = [] {
    const char* e = std::getenv("VR_MMA");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

// Pruned-kernel choice: VR_COOP=1 selects the cooperative warp-per-ray
// kernel instead of the warp-per-32-rays kernel (default).
int vr::coop_mode() {
  static int v = [] {
    const char* e = std::getenv("VR_COOP");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}

// Tensor-core sweep (k_raycast_sweep, d <= 6): VR_SWEEP=1 selects it (read
// per launch, so tests can switch it); off by default -- it is bound by the
// TMEM read rate.
int vr::sweep_mode() {
  const char* e = std::getenv("VR_SWEEP");
  return e ? std::atoi(e) : 0;
}

// mma.sync sweep (k_raycast_hsweep, d <= 6): VR_HSWEEP=1 / 0 (read per launch).
int vr::hsweep_mode() {
  const char* e = std::getenv("VR_HSWEEP");
  return e ? std::atoi(e) : 0;
}

extern "C" int vr_abi_version(void) { return 7; }

extern "C" const char* vr_status_string(int status) {
  switch (status) {
    case VR_OK: return "ok";
    case VR_EINVAL: return "invalid argument";
    case VR_EDIM: return "dimension outside the supported range ([2, 16]; fp32 / pruned paths [2, 8])";
    case VR_ECAPACITY: return "workspace or table capacity exceeded";
    default: break;
  }
  if (status <= VR_ECUDA_BASE) return cudaGetErrorString((cudaError_t)(VR_ECUDA_BASE - status));
  return "unknown status";
}

Screen vr::make_screen(double sqmax, const vr_screen32* s32, int d) {
  Screen sc{};
  sc.fr.sqmax = sqmax;
  if (s32) {
    sc.rec32 = s32->rec;
    sc.rec32p = s32->rec_pairs;
    for (int k = 0; k < VR_MAX_D_ALL; ++k) sc.fr.c0[k] = k < d && k < 8 ? s32->center[k] : 0.0;
    sc.fr.sqmax32 = s32->sqmax;
    sc.fr.bnd32 = s32->bound;
  }
  return sc;
}

extern "C" int vr_record32_stride(int d) {
  if (d < VR_MIN_D || d > VR_MAX_D) return VR_EDIM;
  return rec32_stride(d);
}

extern "C" int vr_record_stride(int d) {
  if (d < VR_MIN_D || d > VR_MAX_D_ALL) return VR_EDIM;
  return rec_stride(d);
}

extern "C" int vr_raycast_batch(const double* rec, int64_t n_gen, int d, double sqmax,
                                const vr_screen32* s32, const double* cand_rec, const int32_t* cand, int64_t n_cand,
                                const double* x, const double* u, const int32_t* eta, int eta_len,
                                int64_t n_rays, int32_t* out_idx, double* out_t, double* out_rp,
                                uint8_t* out_flag, int32_t* recheck_list, int32_t* recheck_count,
                                void* stream) {
  if (!rec || n_gen <= 0 || !x || !u || !eta || !out_idx || !out_t || !out_flag) return VR_EINVAL;
  if (eta_len < 1 || eta_len > d) return VR_EINVAL;
  if ((recheck_list == nullptr) != (recheck_count == nullptr)) return VR_EINVAL;
  const double* crec = cand ? cand_rec : rec;
  const int64_t nc = cand ? n_cand : n_gen;
  if (!crec || nc <= 0) return VR_EINVAL;
  RayOut out{out_idx, out_t, out_rp, out_flag, recheck_list, recheck_count};
  if (d > VR_MAX_D) {
    if (s32) return VR_EDIM;  // fp32 screen: d <= 8
    VR_DISPATCH_D_HIGH(d, {
      SrcExplicit<D> src{x, u, eta, eta_len, rec, n_rays};
      return launch_raycast_fp64<D>(src, n_rays, crec, cand, nc, make_screen(sqmax, nullptr, d),
                                    out, as_stream(stream));
    });
  }
  VR_DISPATCH_D(d, {
    SrcExplicit<D> src{x, u, eta, eta_len, rec, n_rays};
    return launch_raycast<D>(src, n_rays, crec, cand, nc, make_screen(sqmax, s32, d), out,
                             as_stream(stream));
  });
  return VR_OK;
}

extern "C" int vr_raycast_recheck(const double* rec, int64_t n_gen, int d, const double* cand_rec,
                                  const int32_t* cand, int64_t n_cand, const double* x,
                                  const double* u, const int32_t* eta, int eta_len,
                                  const int32_t* recheck_list, const int32_t* recheck_count,
                                  int64_t max_list, int32_t* out_idx, double* out_t,
                                  double* out_rp, uint8_t* out_flag, void* stream) {
  if (!rec || !x || !u || !eta || !recheck_list || !recheck_count) return VR_EINVAL;
  const double* crec = cand ? cand_rec : rec;
  const int64_t nc = cand ? n_cand : n_gen;
  RayOut out{out_idx, out_t, out_rp, out_flag, nullptr, nullptr};
  VR_DISPATCH_D_ALL(d, {
    SrcExplicit<D> src{x, u, eta, eta_len, rec, INT64_MAX};
    return launch_recheck<D>(src, max_list, crec, cand, nc, recheck_list, recheck_count, out,
                             as_stream(stream));
  });
  return VR_OK;
}

extern "C" int vr_raycast_pruned(const double* rec, int64_t n_gen, int d, double sqmax,
                                 const vr_screen32* s32, const vr_prune_index* ix, const double* x, const double* u,
                                 const int32_t* eta, int eta_len, int64_t n_rays,
                                 const int32_t* order, int32_t* out_idx, double* out_t,
                                 double* out_rp, uint8_t* out_flag, int32_t* recheck_list,
                                 int32_t* recheck_count, uint64_t* work, void* stream) {
  if (!rec || !ix || !ix->rec || !ix->perm || !ix->inv_perm || !ix->tile_box || !ix->node_box ||
      !ix->node_range ||
      !x || !u || !eta || !out_idx || !out_t || !out_flag)
    return VR_EINVAL;
  if (eta_len < 1 || eta_len > d || ix->n != n_gen) return VR_EINVAL;
  if ((recheck_list == nullptr) != (recheck_count == nullptr)) return VR_EINVAL;
  RayOut out{out_idx, out_t, out_rp, out_flag, recheck_list, recheck_count};
  const PrunedIndex pi = pruned_index_from(ix, s32 != nullptr);
  const Screen sc = make_screen(sqmax, s32, d);
  VR_DISPATCH_D(d, {
    SrcExplicit<D> src{x, u, eta, eta_len, rec, n_rays, order};
    return launch_raycast_pruned<D>(src, n_rays, pi, sc.fr, out, as_stream(stream),
                                    reinterpret_cast<unsigned long long*>(work));
  });
  return VR_OK;
}

// Processing-order keys / order of a ray batch: csrc/index.cu (vr_ray_keys,
// vr_ray_order).
