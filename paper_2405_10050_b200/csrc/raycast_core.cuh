// Fused rays x generators incircle RayCast.
//
// Reference semantics (pkg/src/voronray/raycast.py:154-224): the converged
// incircle loop returns the valid generator i (u.x_i > thr, raycast.py:95-96,
// 110-117) with the smallest crossing parameter
//     t_i = (|x_i - x|^2 - |x_g - x|^2) / (2 (u.x_i - u.x_g)),   g = eta[0]
// (raycast.py:203; SURVEY.md §8 proves argmin-t == the probe loop).
//
// B200 formulation.  Each thread owns R rays and streams every generator
// through registers; generator tiles are staged in shared memory by TMA bulk
// copies (cp.async.bulk + mbarrier ring).  Instead of evaluating t_i for every
// pair, the kernel keeps the CURRENT best vertex z = x + t_best u and its
// circumsphere radius rho, and runs the incircle test
//     f_i = |x_i|^2 - 2 z.x_i  <  rho^2 - |z|^2                        (*)
// (the power of x_i w.r.t. the current sphere is negative  <=>  t_i < t_best
// for a valid i).  (*) costs one length-d dot product + one FMA per pair,
// i.e. d+2 FP64 pipe ops (2d+2 flops) instead of the 4d+3 of the t form.
// Candidates that pass (*) (or fall inside its rounding band) take the rare
// path: the halfspace test, the reference's centred t formula, and the
// sphere update.  Candidates inside the band +-delta (reference degeneracy
// band 1e-10 plus a rigorous rounding bound) mark the ray RECHECK; such rays
// are re-evaluated exactly by k_raycast_recheck, which also applies the
// reference's runner-up degeneracy test (raycast.py:211-219).
#pragma once

#include "common.cuh"

namespace vr {

// Screening frame: fp64 max |x|^2 for the fp64 rounding bound, and the
// centred fp32 copy's centre / max |x - c|^2 for the fp32 screen's bound.
struct Frame {
  double sqmax;
  double c0[VR_MAX_D_ALL];
  double sqmax32;
  double bnd32;  // max |x_k - c0_k| over generators (fp32 box-test slack)
};

// Candidate records as seen by the kernel: `rec` packed [x, |x|^2, pad].
template <int D>
struct RayState {
  double x[D], u[D];
  double z[D];  // -2 * (x + t_best u): the screening value is |x_i|^2 + z.x_i
  double hi;    // lim + dlt  (screening bound; +inf before the first hit)
  double lim;   // rho^2 - |z|^2 of the current sphere
  double dlt;   // band half-width (degeneracy band + rounding bound)
  double thr;   // halfspace threshold incl. slack
  double s;     // u . x_g
  double base;  // |x - x_g|^2
  double bu;    // u . (x - x_g)
  double tb;    // current best t
  double denb;  // u.(x_best - x_g) of the current best
  double rho2;  // radius^2 of the current sphere (+inf before the first hit)
  float z32[D]; // -2 (z - c0) in fp32 (fp32 screen, centred frame)
  float hi32;   // fp32 screening bound, rounded up, incl. the fp32 error bound
  float u32[D]; // fp32 direction (fp32 box tests)
  float thr32;  // centred halfspace threshold thr - u.c0, rounded down
  float bsl32;  // slack of the fp32 halfspace bound
  float del32;  // slack of the fp32 box distance (centre rounding)
  float rb32;   // (rho^2 + dlt) rounded up with the fp32 sum slack (+inf: none)
  float rbd32;  // (sqrt(rb32) + sqrt(d) del32)^2 rounded up: rb32 with the del32 slack folded in
  float ctc;    // tensor-core screen constant: -(hi32 + tf32 error bound), tf32, rounded down
  int ib;       // current best (local candidate index), -1 = none
  int gk;       // local index of the reference generator g (never valid: u.x_g <= thr), -1 = unknown
  int near;     // 1 -> needs exact re-check
  int nupd;     // sphere updates (work accounting)
#ifdef VR_RARE_STATS
  int st_out, st_self, st_behind, st_band, st_imp;  // rare-path entry outcomes
#endif
};

// tf32 helpers of the tensor-core screen.  tf32_down: the largest tf32 value
// <= v (clears the 13 low mantissa bits toward -inf).
__device__ __forceinline__ float tf32_down(float v) {
  uint32_t b = __float_as_uint(v);
  if (b & 0x1fffu) b = v < 0.0f ? (b & ~0x1fffu) + 0x2000u : (b & ~0x1fffu);
  return __uint_as_float(b);
}
__device__ __forceinline__ uint32_t tf32_rn(float v) {
  uint32_t t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v));
  return t;
}

// Fill the per-ray constants from origin x, direction u and the eta
// generators (global records).  Mirrors _Probe.__init__ (raycast.py:93-96)
// and raycast_incircle's loop constants (raycast.py:178,186-189).
template <int D>
__device__ __forceinline__ void ray_setup(RayState<D>& r, const double* __restrict__ grec,
                                          const int32_t* eta, int eta_len, const Frame& fr) {
  constexpr int S = rec_stride(D);
  const double* xg = grec + (int64_t)eta[0] * S;
  double thr = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) thr = fma(xg[k], r.u[k], thr);
  r.s = thr;
  for (int e = 1; e < eta_len; ++e) {
    const double* xe = grec + (int64_t)eta[e] * S;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) v = fma(xe[k], r.u[k], v);
    thr = fmax(thr, v);
  }
  r.thr = thr + VR_HALFSPACE_SLACK * fmax(1.0, fabs(thr));
  double base = 0.0, bu = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double b = r.x[k] - xg[k];
    base = fma(b, b, base);
    bu = fma(r.u[k], b, bu);
  }
  r.base = base;
  r.bu = bu;
#pragma unroll
  for (int k = 0; k < D; ++k) r.z[k] = -2.0 * r.x[k];
  r.hi = CUDART_INF;
  r.hi32 = CUDART_INF_F;
#pragma unroll
  for (int k = 0; k < D; ++k) r.z32[k] = 0.0f;
  r.lim = CUDART_INF;
  r.dlt = 0.0;
  r.tb = CUDART_INF;
  r.denb = 0.0;
  r.rho2 = CUDART_INF;
  r.ib = -1;
  r.near = 0;
  r.nupd = 0;
#ifdef VR_RARE_STATS
  r.st_out = r.st_self = r.st_behind = r.st_band = r.st_imp = 0;
#endif
  // fp32 box-test constants (centred frame)
  double uc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    r.u32[k] = (float)r.u[k];
    uc = fma(r.u[k], fr.c0[k], uc);
  }
  const double thr_c = r.thr - uc;
  r.thr32 = __double2float_rd(thr_c - 1e-12 * (fabs(thr_c) + fabs(uc) + 1.0));
  r.bsl32 = __double2float_ru((D + 4) * 2.384185791015625e-07 * sqrt((double)D) * fr.bnd32 + 1e-30);
  r.del32 = 0.0f;
  r.rb32 = CUDART_INF_F;
  r.rbd32 = CUDART_INF_F;
  r.ctc = -1e20f;  // no sphere yet: every real candidate passes the tensor-core screen
  r.gk = -1;
}

// Move the screening sphere to the new best crossing t.
template <int D, bool F32>
__device__ __forceinline__ void ray_set_best(RayState<D>& r, double t, double den, int i,
                                             const Frame& fr) {
  const double sqmax = fr.sqmax;
  double zz = 0.0, xx = 0.0, zt2 = 0.0, ztmax = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double zk = fma(t, r.u[k], r.x[k]);  // recomputed bitwise-identically in ray_rare
    if constexpr (!F32) r.z[k] = -2.0 * zk;
    zz = fma(zk, zk, zz);
    xx = fma(r.x[k], r.x[k], xx);
    const double zt = zk - fr.c0[k];
    r.z32[k] = (float)(-2.0 * zt);
    zt2 = fma(zt, zt, zt2);
    ztmax = fmax(ztmax, fabs(zt));
  }
  // Every term of `scale` (and the band) is non-increasing as t decreases
  // (|z(t)|^2 and rho^2(t) are convex in t), so a verdict taken against an
  // older sphere stays conservative for every later one.
  const double tq = t * fma(2.0, fabs(r.bu), fabs(t));
  const double rho2 = fma(t, fma(2.0, r.bu, t), r.base);  // raycast.py:212
  const double scale = fmax(zz, xx) + sqmax + r.base + tq + fabs(rho2);
  const double err = 16.0 * (D + 4) * 2.220446049250313e-16 * scale;
  const double dlt = 2.1e-10 * fmax(r.base, rho2) + err;
  r.lim = rho2 - zz;
  r.dlt = dlt;
  r.hi = r.lim + dlt;
  r.tb = t;
  r.denb = den;
  r.rho2 = rho2;
  r.ib = i;
  ++r.nupd;
  // fp32 screen in the centred frame: |x~|^2 - 2 z~.x~ < rho^2 - |z~|^2 + dlt
  // (+ a bound on the fp32 evaluation error, rounded up), z~ = z - c0.
  const double e32 = 2.0 * (D + 4) * 5.960464477539063e-08 *
                     (fr.sqmax32 + 2.0 * sqrt(zt2 * fr.sqmax32) + 1e-30);
  r.hi32 = __double2float_ru(rho2 - zt2 + dlt + e32);
  // fp32 box test: |e32_k - e_k| <= 2^-22 (|z~|_inf + B); sum slack relative
  r.del32 = __double2float_ru(2.384185791015625e-07 * (ztmax + fr.bnd32));
  r.rb32 = __double2float_ru((rho2 + dlt) * (1.0 + (D + 4) * 1.1920928955078125e-07));
  // The centre / half-extent box tests drop the per-dimension "- del32":
  // with e'_k = max(|z_k - c_k| - h_k, 0) (no slack) and e_k >= max(e'_k -
  // del32, 0), |e| >= |e'| - sqrt(d) del32, so |e'|^2 >= (sqrt(rb32) +
  // sqrt(d) del32)^2 implies |e|^2 >= rb32: the folded test skips a subset of
  // the boxes the per-dimension test skips (del32 ~ 2^-22 of the box scale).
  {
    const float sd = __double2float_ru(sqrt((double)D));
    const float c = __fadd_ru(__fsqrt_ru(r.rb32), __fmul_ru(sd, r.del32));
    r.rbd32 = __fmul_ru(c, c);
  }
  // Tensor-core screen (screen_tile_mma): the same fp32 inputs rounded to
  // tf32 (relative error 2^-11 each, products exact in fp32) and summed by
  // the MMA: |f_tc - f_32| <= 2^-10 sum|z_k x_k| + 2^-11 |x|^2 + accumulation
  // (bounded here by 2^-16 of every term's magnitude), with
  // sum|z_k x_k| <= |z32| |x~|max, |z32|^2 = 4 |z~|^2.  Safety factor 1.25.
  const double sx = sqrt(4.0 * zt2 * fr.sqmax32);
  const double h32 = (double)r.hi32;
  const double etc = 1.25 * (9.765625e-04 * sx + 4.8828125e-04 * fr.sqmax32 +
                             1.52587890625e-05 * (sx + fr.sqmax32 + fabs(h32)));
  r.ctc = tf32_down(__double2float_rd(-(h32 + etc)));
}

template <int D>
__device__ __forceinline__ void load_rec(const double* p, double (&xi)[D]) {
  const double2* p2 = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int k = 0; k < D / 2; ++k) {
    const double2 v = p2[k];
    xi[2 * k] = v.x;
    xi[2 * k + 1] = v.y;
  }
  if (D & 1) xi[D - 1] = p[D - 1];
}

template <int D>
__device__ __forceinline__ float ray_power32(const RayState<D>& r, const float (&xi)[D], float sq) {
  float fp = sq;
#pragma unroll
  for (int k = 0; k < D; ++k) fp = fmaf(r.z32[k], xi[k], fp);
  return fp;
}

template <int D>
__device__ __forceinline__ void load_rec32(const float* p, float (&xi)[D]) {
  const float4* p4 = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int k = 0; k < (D + 3) / 4; ++k) {
    const float4 v = p4[k];
    if (4 * k + 0 < D) xi[4 * k + 0] = v.x;
    if (4 * k + 1 < D) xi[4 * k + 1] = v.y;
    if (4 * k + 2 < D) xi[4 * k + 2] = v.z;
    if (4 * k + 3 < D) xi[4 * k + 3] = v.w;
  }
}

template <int D>
__device__ __forceinline__ void load_rec_g(const double* p, double (&xi)[D]) {
  const double2* p2 = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int k = 0; k < D / 2; ++k) {
    const double2 v = __ldg(p2 + k);
    xi[2 * k] = v.x;
    xi[2 * k + 1] = v.y;
  }
  if (D & 1) xi[D - 1] = __ldg(p + D - 1);
}

// Block-batched rare path for one ray: the candidates of one 8-candidate
// block that passed the (conservative) screen, in index order.  Equivalent to
// processing them one by one with immediate sphere updates: the final sphere
// is that of the improving candidate with the smallest t (division-free
// comparison, first index on exact ties), a single update; every other
// improving candidate is re-tested against the new sphere and flags RECHECK
// if it lies inside the new band; the previous best is tested as before.
template <int D, bool F32>
__device__ __forceinline__ void ray_rare_block(RayState<D>& r, const double* tile, unsigned mm,
                                               int gbase, const Frame& fr) {
  constexpr int S = rec_stride(D);
  const bool have0 = r.ib >= 0;
  double zk2[D];
#pragma unroll
  for (int k = 0; k < D; ++k)
    zk2[k] = F32 ? (have0 ? -2.0 * fma(r.tb, r.u[k], r.x[k]) : 0.0) : r.z[k];
  double bn = 0.0, bd = 0.0;
  int bu = -1;
  unsigned imp = 0u;
  while (mm) {
    const int u = __ffs(mm) - 1;
    mm &= mm - 1;
    double xi[D];
    load_rec<D>(tile + u * S, xi);
    double fp = tile[u * S + D], q = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      fp = fma(zk2[k], xi[k], fp);
      q = fma(r.u[k], xi[k], q);
    }
#ifdef VR_RARE_STATS
#define VR_ST(f) ++r.f
#else
#define VR_ST(f) (void)0
#endif
    if (have0 && !(fp < r.hi)) { VR_ST(st_out); continue; }  // outside the block-start band
    if (gbase + u == r.ib) { VR_ST(st_self); continue; }     // the current best itself
    if (!(q > r.thr)) { VR_ST(st_behind); continue; }        // behind the halfspace (raycast.py:110-117)
    if (have0 && fp >= r.lim - r.dlt) r.near = 1;
    if (have0 && !(fp < r.lim)) { VR_ST(st_band); continue; }
    VR_ST(st_imp);
#undef VR_ST
    double aa = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double a = r.x[k] - xi[k];
      aa = fma(a, a, aa);
    }
    const double num = aa - r.base, den = q - r.s;  // raycast.py:201-203
    if (bu < 0 || num * bd < bn * den) { bn = num; bd = den; bu = u; }
    imp |= 1u << u;
  }
  if (bu < 0) return;
  const double t = bn / (2.0 * bd);
  const double told = r.tb, denold = r.denb;
  ray_set_best<D, F32>(r, t, bd, gbase + bu, fr);
  if (have0 && 2.0 * denold * (told - t) < r.dlt) r.near = 1;
  imp &= ~(1u << bu);
  if (imp) {
#pragma unroll
    for (int k = 0; k < D; ++k) zk2[k] = -2.0 * fma(t, r.u[k], r.x[k]);
    while (imp) {
      const int u = __ffs(imp) - 1;
      imp &= imp - 1;
      double xi[D];
      load_rec<D>(tile + u * S, xi);
      double fp = tile[u * S + D];
#pragma unroll
      for (int k = 0; k < D; ++k) fp = fma(zk2[k], xi[k], fp);
      if (fp < r.hi) r.near = 1;  // in the new sphere's band (it has t >= t_new)
    }
  }
}

// Screening value of one pair: |x_i|^2 - 2 z.x_i as one chain of d FMAs
// (z is stored pre-scaled by -2), so a pair costs d DFMA + 1 DSETP.
template <int D>
__device__ __forceinline__ double ray_power(const RayState<D>& r, const double (&xi)[D],
                                            double sq) {
  double fp = sq;
#pragma unroll
  for (int k = 0; k < D; ++k) fp = fma(r.z[k], xi[k], fp);
  return fp;
}

// ---------------------------------------------------------------------------
// Ray sources.  load() fills x, u and calls ray_setup; returns false for
// padding lanes (k >= n).
// ---------------------------------------------------------------------------
template <int D>
struct SrcExplicit {
  const double* x;
  const double* u;
  const int32_t* eta;
  int eta_len;
  const double* grec;
  int64_t n;
  const int32_t* order = nullptr;  // optional processing order (slot -> ray id)
  __device__ __forceinline__ int64_t id(int64_t k) const { return order ? order[k] : k; }
  __device__ __forceinline__ int32_t gen(int64_t k) const { return eta[id(k) * eta_len]; }
  __host__ __device__ __forceinline__ int eta_count() const { return eta_len; }
  __device__ __forceinline__ int32_t eta_at(int64_t k, int e) const { return eta[id(k) * eta_len + e]; }
  __device__ __forceinline__ bool load(int64_t k, RayState<D>& r, const Frame& fr) const {
    if (k >= n) return false;
    k = id(k);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      r.x[j] = x[k * D + j];
      r.u[j] = u[k * D + j];
    }
    ray_setup<D>(r, grec, eta + k * eta_len, eta_len, fr);
    return true;
  }
};

// Philox4x32-10 (Salmon et al. 2011) -- counter-based, so every (seed, cell,
// ray) direction is independent of the launch shape and of the GPU count.
__device__ __forceinline__ void philox4x32_10(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int rnd = 0; rnd < 10; ++rnd) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// D standard normals for ray `ray` of generator `cell`: Philox counter
// (ray, cell, pair, 0x4D43), Box-Muller on 53-bit uniforms.
template <int D>
__device__ __forceinline__ void philox_normals(uint64_t seed, int64_t cell, int64_t ray,
                                               double (&z)[D]) {
#pragma unroll
  for (int p = 0; p < (D + 1) / 2; ++p) {
    uint32_t c[4] = {(uint32_t)ray, (uint32_t)cell, (uint32_t)p | ((uint32_t)(ray >> 32) << 8),
                     0x4D430000u | (uint32_t)((cell >> 32) & 0xFFFF)};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint64_t a = ((((uint64_t)c[0]) << 32) | c[1]) >> 11;
    const uint64_t b = ((((uint64_t)c[2]) << 32) | c[3]) >> 11;
    const double u1 = (double)(a + 1) * 0x1.0p-53;  // (0, 1]
    const double u2 = (double)b * 0x1.0p-53;        // [0, 1)
    const double rad = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos(6.283185307179586 * u2, &sn, &cs);
    z[2 * p] = rad * cs;
    if (2 * p + 1 < D) z[2 * p + 1] = rad * sn;
  }
}

// Unit direction exactly as sample_unit_sphere (integrate_mc.py:51-56):
// y = z / sqrt(z.z).
template <int D>
__device__ __forceinline__ void normalise(const double (&z)[D], double (&y)[D]) {
  double zz = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) zz = fma(z[k], z[k], zz);
  const double nrm = sqrt(zz);
#pragma unroll
  for (int k = 0; k < D; ++k) y[k] = z[k] / nrm;
}

template <int D>
struct SrcMC {
  const double* grec;
  const int32_t* cells;
  int64_t per;    // rays per cell
  const double* dirs;  // nullable: raw Gaussian draws (n, D)
  uint64_t seed;
  int64_t n;      // total rays
  const int32_t* order = nullptr;  // optional processing order (slot -> ray id)
  __device__ __forceinline__ void direction(int64_t k, double (&y)[D]) const {
    double z[D];
    if (dirs) {
#pragma unroll
      for (int j = 0; j < D; ++j) z[j] = dirs[k * D + j];
    } else {
      const int64_t c = k / per;
      philox_normals<D>(seed, cells[c], k - c * per, z);
    }
    normalise<D>(z, y);
  }
  __device__ __forceinline__ int64_t id(int64_t k) const { return order ? order[k] : k; }
  __device__ __forceinline__ int32_t gen(int64_t k) const { return cells[id(k) / per]; }
  __host__ __device__ __forceinline__ int eta_count() const { return 1; }
  __device__ __forceinline__ int32_t eta_at(int64_t k, int) const { return gen(k); }
  __device__ __forceinline__ bool load(int64_t k, RayState<D>& r, const Frame& fr) const {
    if (k >= n) return false;
    k = id(k);
    const int32_t cell = cells[k / per];
    const double* xc = grec + (int64_t)cell * rec_stride(D);
#pragma unroll
    for (int j = 0; j < D; ++j) r.x[j] = xc[j];
    direction(k, r.u);
    ray_setup<D>(r, grec, &cell, 1, fr);
    return true;
  }
};

// ---------------------------------------------------------------------------
// Outputs.
// ---------------------------------------------------------------------------
struct RayOut {
  int32_t* idx;
  double* t;
  double* rp;  // nullable
  uint8_t* flag;
  int32_t* recheck_list;   // nullable
  int32_t* recheck_count;  // nullable
};

template <int D>
__device__ __forceinline__ void ray_store(const RayState<D>& r, int64_t k,
                                          const int32_t* __restrict__ cand, const RayOut& o) {
  if (r.ib < 0) {
    o.idx[k] = -1;
    o.t[k] = CUDART_INF;
    o.flag[k] = VR_RAY_ESCAPED;
    if (o.rp) {
#pragma unroll
      for (int j = 0; j < D; ++j) o.rp[k * D + j] = CUDART_NAN;
    }
    return;
  }
  o.idx[k] = cand ? cand[r.ib] : r.ib;
  o.t[k] = r.tb;
  if (o.rp) {
#pragma unroll
    for (int j = 0; j < D; ++j) o.rp[k * D + j] = fma(r.tb, r.u[j], r.x[j]);  // raycast.py:210
  }
  if (r.near) {
    o.flag[k] = VR_RAY_RECHECK;
    if (o.recheck_list) {
      int slot = atomicAdd(o.recheck_count, 1);
      o.recheck_list[slot] = (int32_t)k;
    }
  } else {
    o.flag[k] = VR_RAY_OK;
  }
}

// ---------------------------------------------------------------------------
// Screening of one tile (PT records) for the R rays of every lane: blocks of
// U=8 candidates x R rays of independent dot products (fp32 in the centred
// frame when F32, else fp64), per-ray bitmasks, one warp vote per block,
// then the in-order fp64 rare path.  The screen is conservative (stale-safe:
// a candidate outside an older sphere is outside every later one; the fp32
// bound covers the fp32 evaluation error), and the fp64 rare path re-applies
// the exact fp64 test first, so the result is independent of F32.
// ---------------------------------------------------------------------------
struct WarpCounters {
  unsigned long long rare_blocks = 0, rare_iters = 0, entries = 0;
};

template <int D, int R, int PT, bool F32>
__device__ __forceinline__ void screen_tile(RayState<D> (&ray)[R], const double* tile,
                                            const float* tile32, int gbase, const Frame& fr,
                                            WarpCounters* wc = nullptr) {
  constexpr int S = rec_stride(D);
  constexpr int S32 = rec32_stride(D);
  constexpr int U = 8;
  for (int c = 0; c < PT; c += U) {
    unsigned m[R];
#pragma unroll
    for (int j = 0; j < R; ++j) m[j] = 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (F32) {
        float xi[D];
        load_rec32<D>(tile32 + (c + u) * S32, xi);
        const float sq = tile32[(c + u) * S32 + D];
#pragma unroll
        for (int j = 0; j < R; ++j)
          m[j] |= (ray_power32<D>(ray[j], xi, sq) < ray[j].hi32) ? (1u << u) : 0u;
      } else {
        double xi[D];
        load_rec<D>(tile + (c + u) * S, xi);
        const double sq = tile[(c + u) * S + D];
#pragma unroll
        for (int j = 0; j < R; ++j)
          m[j] |= (ray_power<D>(ray[j], xi, sq) < ray[j].hi) ? (1u << u) : 0u;
      }
    }
    unsigned any = 0u;
#pragma unroll
    for (int j = 0; j < R; ++j) any |= m[j];
    if (__any_sync(0xffffffffu, any != 0u)) {
      if constexpr (F32) {
        // conservative fp32 halfspace pre-filter + the current best itself
        // (most screen hits of a stale sphere lie behind the ray)
#pragma unroll
        for (int j = 0; j < R; ++j) {
          unsigned mm = m[j], h = 0u;
          while (mm) {
            const int u = __ffs(mm) - 1;
            mm &= mm - 1;
            float xi[D];
            load_rec32<D>(tile32 + (c + u) * S32, xi);
            float q = ray[j].bsl32;
#pragma unroll
            for (int k = 0; k < D; ++k) q = fmaf(ray[j].u32[k], xi[k], q);
            if (q > ray[j].thr32 && gbase + c + u != ray[j].ib) h |= 1u << u;
          }
          m[j] = h;
        }
      }
      if (wc) {
        ++wc->rare_blocks;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          wc->entries += __popc(m[j]);
          wc->rare_iters += __reduce_max_sync(0xffffffffu, (unsigned)__popc(m[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (m[j]) ray_rare_block<D, F32>(ray[j], tile + c * S, m[j], gbase + c, fr);
    }
  }
}

#ifndef VR_PAIR_BLOCK
#define VR_PAIR_BLOCK 16
#endif

// Packed fp32 pairs (sm_100 FFMA2: two IEEE fp32 FMAs per instruction; a
// scalar multiplicand is broadcast by ptxas, so z32 needs no duplication).
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// screen_tile over the pair-interleaved fp32 layout (rec32p_stride): the same
// per-pair values as ray_power32 (same FMA order, IEEE fp32 per lane), two
// candidates per FFMA2; the block vote is taken on the minimum (one FMNMX per
// candidate), and the per-candidate mask is built only when the vote fires.
template <int D, int R, int PT>
__device__ __forceinline__ void screen_tile_pairs(RayState<D> (&ray)[R], const double* tile,
                                                  const float* tilep, int gbase, const Frame& fr,
                                                  WarpCounters* wc = nullptr) {
  constexpr int S = rec_stride(D);
  constexpr int P2 = rec32p_stride(D);
  constexpr int U = VR_PAIR_BLOCK;
  for (int c = 0; c < PT; c += U) {
    float f[R][U];
#pragma unroll
    for (int p = 0; p < U / 2; ++p) {
      const float4* q = reinterpret_cast<const float4*>(tilep + ((c >> 1) + p) * P2);
      float v[P2];
#pragma unroll
      for (int k = 0; k < P2 / 4; ++k) {
        const float4 w = q[k];
        v[4 * k] = w.x;
        v[4 * k + 1] = w.y;
        v[4 * k + 2] = w.z;
        v[4 * k + 3] = w.w;
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        uint64_t acc = f2pack(v[2 * D], v[2 * D + 1]);
#pragma unroll
        for (int k = 0; k < D; ++k)
          acc = ffma2(f2pack(ray[j].z32[k], ray[j].z32[k]), f2pack(v[2 * k], v[2 * k + 1]), acc);
        f2unpack(acc, f[j][2 * p], f[j][2 * p + 1]);
      }
    }
    bool any = false;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      // pairwise (tree) minimum: log2(U) dependent steps instead of U - 1
      float t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) t[u] = f[j][u];
#pragma unroll
      for (int w = U / 2; w >= 1; w /= 2) {
#pragma unroll
        for (int u = 0; u < w; ++u) t[u] = fminf(t[u], t[u + w]);
      }
      any |= t[0] < ray[j].hi32;
    }
    if (__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        unsigned m = 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) m |= (f[j][u] < ray[j].hi32) ? (1u << u) : 0u;
        // fp32 halfspace pre-filter (conservative, the box tests' bound): most
        // candidates inside the stale sphere lie behind the ray's halfspace
        // and would be rejected by the fp64 rare path anyway (raycast.py:110-117).
        if (__any_sync(0xffffffffu, m != 0u)) {
          unsigned h = 0u;
#pragma unroll 1
          for (int p = 0; p < U / 2; ++p) {
            const float4* q = reinterpret_cast<const float4*>(tilep + ((c >> 1) + p) * P2);
            float v[P2];
#pragma unroll
            for (int k = 0; k < P2 / 4; ++k) {
              const float4 w = q[k];
              v[4 * k] = w.x;
              v[4 * k + 1] = w.y;
              v[4 * k + 2] = w.z;
              v[4 * k + 3] = w.w;
            }
            uint64_t acc = f2pack(ray[j].bsl32, ray[j].bsl32);
#pragma unroll
            for (int k = 0; k < D; ++k)
              acc = ffma2(f2pack(ray[j].u32[k], ray[j].u32[k]), f2pack(v[2 * k], v[2 * k + 1]), acc);
            float qa, qb;
            f2unpack(acc, qa, qb);
            h |= (qa > ray[j].thr32 ? 1u : 0u) << (2 * p);
            h |= (qb > ray[j].thr32 ? 1u : 0u) << (2 * p + 1);
          }
          m &= h;
          const int rel = ray[j].ib - (gbase + c);  // the current best itself
          if ((unsigned)rel < (unsigned)U) m &= ~(1u << rel);
        }
        if (wc) {
          if (j == 0) ++wc->rare_blocks;
          wc->entries += __popc(m);
          wc->rare_iters += __reduce_max_sync(0xffffffffu, (unsigned)__popc(m));
        }
        if (m) ray_rare_block<D, true>(ray[j], tile + c * S, m, gbase + c, fr);
      }
    }
  }
}

template <int D, int R>
__device__ __forceinline__ void init_padding_lane(RayState<D>& r) {
  r.hi = -CUDART_INF;
  r.hi32 = -CUDART_INF_F;
  r.thr = CUDART_INF;  // never needs a box
  r.thr32 = CUDART_INF_F;
  r.bsl32 = 0.0f;
  r.ctc = 1e30f;  // never passes the tensor-core screen
  r.ib = -1;
  r.gk = -1;
#pragma unroll
  for (int k = 0; k < D; ++k) r.u32[k] = 0.0f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    r.z[k] = 0.0;
    r.z32[k] = 0.0f;
  }
}

// ---------------------------------------------------------------------------
// Exhaustive kernel: NT threads x R rays; every generator tile goes through a
// STAGES-deep shared-memory ring filled by TMA bulk copies (fp64 records, plus
// the centred fp32 copy when F32); the last warp to release a stage issues
// its refill.
// ---------------------------------------------------------------------------
template <int D, int R, int NT, int TILE, int STAGES, int MINB, bool F32, class Src,
          bool PAIRS = false>
__global__ void __launch_bounds__(NT, MINB)
    k_raycast(Src src, const double* __restrict__ crec, const float* __restrict__ crec32,
              const int32_t* __restrict__ cand, int64_t n_cand, Frame fr, RayOut out) {
  constexpr int S = rec_stride(D);
  // fp32 rows: row layout (S32 floats per record) or pair-interleaved (P2
  // floats per two records, packed FFMA2 screen)
  constexpr int S32 = PAIRS ? rec32p_stride(D) : rec32_stride(D);
  constexpr int F32_PER_TILE = PAIRS ? TILE / 2 * S32 : TILE * S32;
  constexpr int NW = NT / 32;
  static_assert(TILE % 16 == 0 && VR_REC_PAD % TILE == 0, "tile must divide the record padding");
  static_assert(!PAIRS || F32, "pairs are an fp32 layout");
  constexpr uint32_t BYTES64 = (uint32_t)(TILE * S * sizeof(double));
  constexpr uint32_t BYTES32 = F32 ? (uint32_t)(F32_PER_TILE * sizeof(float)) : 0u;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* tiles = reinterpret_cast<double*>(smem_raw);
  float* tiles32 = reinterpret_cast<float*>(smem_raw + (size_t)STAGES * BYTES64);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)STAGES * (BYTES64 + BYTES32));
  int* released = reinterpret_cast<int*>(full + STAGES);

  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t ntiles = (n_cand + TILE - 1) / TILE;
  auto issue = [&](int64_t t) {
    const int st = (int)(t % STAGES);
    mbar_arrive_expect_tx(&full[st], BYTES64 + BYTES32);
    bulk_g2s(tiles + (size_t)st * TILE * S, crec + t * TILE * S, BYTES64, &full[st]);
    if constexpr (F32)
      bulk_g2s(tiles32 + (size_t)st * F32_PER_TILE, crec32 + t * F32_PER_TILE, BYTES32, &full[st]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int64_t t = 0; t < ntiles && t < STAGES; ++t) issue(t);
  }

  RayState<D> ray[R];
  bool act[R];
  const int64_t k0 = (int64_t)blockIdx.x * NT * R + tid;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    act[j] = src.load(k0 + (int64_t)j * NT, ray[j], fr);
    if (!act[j]) init_padding_lane<D, R>(ray[j]);
  }

  for (int64_t t = 0; t < ntiles; ++t) {
    const int st = (int)(t % STAGES);
    mbar_wait(&full[st], (uint32_t)((t / STAGES) & 1));
    if constexpr (PAIRS)
      screen_tile_pairs<D, R, TILE>(ray, tiles + (size_t)st * TILE * S,
                                    tiles32 + (size_t)st * F32_PER_TILE, (int)(t * TILE), fr);
    else
      screen_tile<D, R, TILE, F32>(ray, tiles + (size_t)st * TILE * S,
                                   tiles32 + (size_t)st * F32_PER_TILE, (int)(t * TILE), fr);
    // release the stage; the last warp to release it issues the refill
    __syncwarp();
    if (lane == 0) {
      const int old = atomicAdd(&released[st], 1);
      if (old == NW - 1) {
        released[st] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (t + STAGES < ntiles) issue(t + STAGES);
      }
    }
  }

#pragma unroll
  for (int j = 0; j < R; ++j)
    if (act[j]) ray_store<D>(ray[j], src.id(k0 + (int64_t)j * NT), cand, out);
}

// ---------------------------------------------------------------------------
// Pruned RayCast: generators in kd-order, grouped in
// tiles of PT records with axis-aligned bounding boxes, tiles grouped in
// blocks of PB tiles with their own boxes.  A warp (32 lanes x R rays,
// spatially coherent) skips a block / tile when for EVERY ray of the warp the
// box is either entirely behind the ray's halfspace or certifiably outside
// its current sphere plus band -- such a tile holds no candidate that could
// improve the ray or fall in its degeneracy band, now or for any later
// (smaller) sphere.  Everything not skipped goes through exactly the same
// screening / rare path as the exhaustive kernel, so results are identical.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ bool ray_needs_box(const RayState<D>& r, const double* __restrict__ box) {
  // box = [lo_0..lo_{D-1}, hi_0..hi_{D-1}]
  double umax = 0.0, d2 = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double lo = __ldg(box + k), hi = __ldg(box + D + k);
    umax = fma(r.u[k], r.u[k] > 0.0 ? hi : lo, umax);
    const double zc = -0.5 * r.z[k];
    const double e = fmax(fmax(lo - zc, zc - hi), 0.0);
    d2 = fma(e, e, d2);
  }
  // every candidate of the box is behind the forward halfspace
  if (umax + 1e-13 * (fabs(umax) + 1.0) <= r.thr) return false;
  if (r.ib < 0) return true;  // no sphere yet
  // power of any box point w.r.t. the sphere >= d2 - rho2
  return d2 < r.rho2 + r.dlt + 1e-12 * (r.rho2 + d2);
}

// fp32 box test in the centred frame (boxes rounded outward on the host):
// skip only if the fp32 bounds certify "behind the halfspace" or "outside the
// sphere + band" for the exact box.  box32 = [lo_0..lo_{D-1}, hi_0..hi_{D-1}].
// fp32 box records: [lo_0..lo_{D-1}, hi_0..hi_{D-1}] padded to a multiple
// of 4 floats (16-B rows, loaded as float4).
__host__ __device__ constexpr int box32_stride(int d) { return (2 * d + 3) & ~3; }

template <int D>
__device__ __forceinline__ bool ray_needs_box32(const RayState<D>& r,
                                                const float* __restrict__ box) {
  constexpr int BS = box32_stride(D);
  float v[BS];
  const float4* b4 = reinterpret_cast<const float4*>(box);
#pragma unroll
  for (int k = 0; k < BS / 4; ++k) {
    const float4 w = __ldg(b4 + k);
    v[4 * k] = w.x;
    v[4 * k + 1] = w.y;
    v[4 * k + 2] = w.z;
    v[4 * k + 3] = w.w;
  }
  float lo[D], hi[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    lo[k] = v[k];
    hi[k] = v[D + k];
  }
  float umax = 0.0f, d2 = 0.0f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    umax = fmaf(r.u32[k], r.u32[k] > 0.0f ? hi[k] : lo[k], umax);
    const float zc = -0.5f * r.z32[k];
    const float e = fmaxf(fmaxf(lo[k] - zc, zc - hi[k]) - r.del32, 0.0f);
    d2 = fmaf(e, e, d2);
  }
  if (umax + r.bsl32 <= r.thr32) return false;  // behind the forward halfspace
  return !(d2 >= r.rb32);                        // inside sphere + band (or no sphere)
}

// The same test on centre / half-extent rows [c_0..c_{D-1}, h_0..h_{D-1}]
// (vr_prune_index.node_cb32; [c - h, c + h] contains the exact box): the
// halfspace maximum is sum u_k c_k + |u_k| h_k and the distance term
// max(|z_k - c_k| - h_k, 0) -- 7 instead of 9 instructions per dimension.
// Rounding: |c| + h <= B, so both evaluations stay within the del32 / bsl32
// slacks derived for the [lo, hi] form.
template <int D>
__device__ __forceinline__ bool ray_needs_box32_ch(const RayState<D>& r,
                                                   const float* __restrict__ box) {
  constexpr int BS = box32_stride(D);
  float v[BS];
  const float4* b4 = reinterpret_cast<const float4*>(box);
#pragma unroll
  for (int k = 0; k < BS / 4; ++k) {
    const float4 w = __ldg(b4 + k);
    v[4 * k] = w.x;
    v[4 * k + 1] = w.y;
    v[4 * k + 2] = w.z;
    v[4 * k + 3] = w.w;
  }
  float umax = 0.0f, d2 = 0.0f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    umax = fmaf(r.u32[k], v[k], umax);
    umax = fmaf(fabsf(r.u32[k]), v[D + k], umax);
    const float zc = -0.5f * r.z32[k];
#ifdef VR_NO_FOLD_DEL
    const float e = fmaxf(fabsf(zc - v[k]) - v[D + k] - r.del32, 0.0f);
#else
    const float e = fmaxf(fabsf(zc - v[k]) - v[D + k], 0.0f);  // del32 folded into rbd32
#endif
    d2 = fmaf(e, e, d2);
  }
  if (umax + r.bsl32 <= r.thr32) return false;  // behind the forward halfspace
#ifdef VR_NO_FOLD_DEL
  return !(d2 >= r.rb32);                        // inside sphere + band (or no sphere)
#else
  return !(d2 >= r.rbd32);
#endif
}

// ray_needs_box32_ch plus the sphere-distance term d2 (child ordering).
template <int D>
__device__ __forceinline__ bool ray_needs_box32_ch_d2(const RayState<D>& r,
                                                      const float* __restrict__ box, float& d2) {
  constexpr int BS = box32_stride(D);
  float v[BS];
  const float4* b4 = reinterpret_cast<const float4*>(box);
#pragma unroll
  for (int k = 0; k < BS / 4; ++k) {
    const float4 w = __ldg(b4 + k);
    v[4 * k] = w.x;
    v[4 * k + 1] = w.y;
    v[4 * k + 2] = w.z;
    v[4 * k + 3] = w.w;
  }
  float umax = 0.0f;
  d2 = 0.0f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    umax = fmaf(r.u32[k], v[k], umax);
    umax = fmaf(fabsf(r.u32[k]), v[D + k], umax);
    const float zc = -0.5f * r.z32[k];
#ifdef VR_NO_FOLD_DEL
    const float e = fmaxf(fabsf(zc - v[k]) - v[D + k] - r.del32, 0.0f);
#else
    const float e = fmaxf(fabsf(zc - v[k]) - v[D + k], 0.0f);
#endif
    d2 = fmaf(e, e, d2);
  }
  if (umax + r.bsl32 <= r.thr32) return false;
#ifdef VR_NO_FOLD_DEL
  return !(d2 >= r.rb32);
#else
  return !(d2 >= r.rbd32);
#endif
}

template <int D, bool F32, bool CH = false>
__device__ __forceinline__ bool ray_needs(const RayState<D>& r, const double* __restrict__ box64,
                                          const float* __restrict__ box32, int64_t b) {
  if constexpr (F32 && CH) return ray_needs_box32_ch<D>(r, box32 + b * box32_stride(D));
  else if constexpr (F32) return ray_needs_box32<D>(r, box32 + b * box32_stride(D));
  else return ray_needs_box<D>(r, box64 + b * 2 * D);
}

// Seed pass: the valid candidate with the smallest t in one tile, found
// without divergence (division-free comparison num_i den_b < num_b den_i,
// den > 0), then one sphere update.  Purely an accelerator: the main scan
// screens the seed tile again, so near-ties / rounding in the seed choice are
// caught by the regular rare path (update or RECHECK flag).
template <int D, int R, int PT, bool F32>
__device__ __forceinline__ void seed_tile(RayState<D> (&ray)[R], const double* __restrict__ tile,
                                          int gbase, const Frame& fr) {
  constexpr int S = rec_stride(D);
  double nb[R], db[R];
  int ib[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    nb[j] = 1.0;
    db[j] = 0.0;  // "t = +inf"
    ib[j] = -1;
  }
#pragma unroll 2
  for (int c = 0; c < PT; ++c) {
    double xi[D];
    load_rec_g<D>(tile + c * S, xi);
    const bool real = !isinf(__ldg(tile + c * S + D));
#pragma unroll
    for (int j = 0; j < R; ++j) {
      double q = 0.0, aa = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        q = fma(ray[j].u[k], xi[k], q);
        const double a = ray[j].x[k] - xi[k];
        aa = fma(a, a, aa);
      }
      const double num = aa - ray[j].base, den = q - ray[j].s;
      const bool better = real && q > ray[j].thr && num * db[j] < nb[j] * den;
      nb[j] = better ? num : nb[j];
      db[j] = better ? den : db[j];
      ib[j] = better ? gbase + c : ib[j];
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (ib[j] < 0) continue;
    const double t = nb[j] / (2.0 * db[j]);
    if (ray[j].ib < 0 || t < ray[j].tb) ray_set_best<D, F32>(ray[j], t, db[j], ib[j], fr);
  }
}

// fp32 seed pass (tensor-core kernel): the same division-free argmin over
// the start tile, evaluated on the centred fp32 rows (broadcast loads, 4
// candidates in flight) with the conservative fp32 halfspace test; only the
// winner is re-evaluated in fp64 (reference formula, raycast.py:201-203) and
// must pass the exact halfspace test before it seeds the sphere.  Like the
// fp64 seed it is purely an accelerator: the main scan screens the seed tile
// again, so a suboptimal (or skipped) seed never changes a result.
template <int D>
__device__ __forceinline__ void seed_tile32(RayState<D>& r, const float* __restrict__ tile32,
                                            const double* __restrict__ tile64, int gbase,
                                            const Frame& fr) {
  constexpr int S = rec_stride(D);
  constexpr int S32 = rec32_stride(D);
  float xo[D];
  double uc = 0.0, xx = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    xo[k] = (float)(r.x[k] - fr.c0[k]);
    uc = fma(r.u[k], fr.c0[k], uc);
    xx = fma((double)xo[k], (double)xo[k], xx);
  }
  const float base = (float)r.base, sc = (float)(r.s - uc);
  // The eta generators (equidistant to x: num ~ 0) pass the conservative
  // fp32 halfspace test and would win with t ~ 0; real candidates have
  // num > 0 by the empty sphere of the origin vertex.  Skip num below a bound
  // on the fp32 error of |x~ - x~_i|^2 - base (seed quality only).
  const float nmin = (float)(16.0 * D * 5.960464477539063e-08 * (2.0 * fr.sqmax32 + 2.0 * xx + r.base));
  const int gl = r.gk - gbase;
  float nb = 1.0f, db = 0.0f;  // "t = +inf"
  int ib = -1;
#ifndef VR_SEED_UNROLL
#define VR_SEED_UNROLL 4
#endif
  constexpr int SEED_UNROLL = VR_SEED_UNROLL;
#pragma unroll SEED_UNROLL
  for (int c = 0; c < 64; ++c) {
    float xi[D];
    load_rec32<D>(tile32 + c * S32, xi);
    const float sq = __ldg(tile32 + c * S32 + D);
    float q = r.bsl32, aa = 0.0f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      q = fmaf(r.u32[k], xi[k], q);
      const float a = xo[k] - xi[k];
      aa = fmaf(a, a, aa);
    }
    const float num = aa - base, den = q - r.bsl32 - sc;
    const bool better = !isinf(sq) && c != gl && q > r.thr32 && den > 0.0f && num > nmin &&
                        num * db < nb * den;
    nb = better ? num : nb;
    db = better ? den : db;
    ib = better ? c : ib;
  }
  if (ib < 0) return;
  double xi[D];
  load_rec_g<D>(tile64 + ib * S, xi);
  double q = 0.0, aa = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    q = fma(r.u[k], xi[k], q);
    const double a = r.x[k] - xi[k];
    aa = fma(a, a, aa);
  }
  if (!(q > r.thr)) return;  // the fp32 choice was not valid
  const double num = aa - r.base, den = q - r.s;
  const double t = num / (2.0 * den);
  if (r.ib < 0 || t < r.tb) ray_set_best<D, true>(r, t, den, gbase + ib, fr);
}

// Warp-coherent traversal of the kd tree over tiles (heap layout: node i has
// children 2i+1, 2i+2; node_range[i] = [first tile, last tile + 1); a leaf is
// one tile).  A node is descended only if some ray of the warp needs its box
// (halfspace + current sphere + band); children are pushed so that the one
// holding the warp's start tile is visited first.
template <int D, int R, bool F32, bool CH = false>
struct TreeCursor {
  // Warp-distributed stack: slot i lives in lane i's registers (push = one
  // lane writes, pop = shuffle), so the DFS touches no local memory.  The DFS
  // holds at most depth + 1 <= 32 entries for trees of < 2^31 tiles.  Each
  // entry keeps the lanes whose rays needed the node when it was pushed
  // (spheres only shrink, so the mask stays a superset of the later need).
  int s_node = 0, s_lo = 0, s_hi = 0;
  unsigned s_mask = 0u;
  int sp = 0;
  int64_t st = 0;
  unsigned long long tests = 0;
  unsigned leaf_mask = 0u;  // lanes needing the leaf returned by next()
  int pend = 0, pend_end = 0;  // rest of a popped multi-tile leaf (VR_LEAF_TILES > 1)
  __device__ __forceinline__ unsigned warp_needs(const RayState<D> (&ray)[R],
                                                 const double* __restrict__ node_box,
                                                 const float* __restrict__ node_box32, int node) {
    bool need = false;
#pragma unroll
    for (int j = 0; j < R; ++j) need |= ray_needs<D, F32, CH>(ray[j], node_box, node_box32, node);
    ++tests;
    return __ballot_sync(0xffffffffu, need);
  }
  __device__ __forceinline__ void push(int node, int2 rg, unsigned m) {
    if (sp >= 32) __trap();
    if ((int)(threadIdx.x & 31) == sp) {
      s_node = node;
      s_lo = rg.x;
      s_hi = rg.y;
      s_mask = m;
    }
    ++sp;
  }
  __device__ __forceinline__ void init(int64_t start_tile, const RayState<D> (&ray)[R],
                                       const double* __restrict__ node_box,
                                       const float* __restrict__ node_box32,
                                       const int2* __restrict__ node_range) {
    st = start_tile;
    sp = 0;
    pend = pend_end = 0;
    const unsigned m = warp_needs(ray, node_box, node_box32, 0);
    if (m) push(0, __ldg(node_range), m);
  }
  // Children are tested when their parent is expanded (both boxes loaded
  // together, one dependent step per level); a popped leaf is returned.
  __device__ __forceinline__ int64_t next(const RayState<D> (&ray)[R],
                                          const double* __restrict__ node_box,
                                          const float* __restrict__ node_box32,
                                          const int2* __restrict__ node_range) {
    // Nodes of <= LT tiles are screened whole (their children are not
    // box-tested).  At d >= 7 the walk costs more than the screens it saves:
    // LT = 2 takes config 5 from 0.787 to 0.767 s (1,515 instead of 2,212 node
    // tests, 724 instead of 528 tiles per warp of edge rays); at d <= 6 it is
    // neutral (config 2: 2.416 vs 2.430 ms) or slower (config 4: 0.081 vs
    // 0.079 s).  -DVR_LEAF_TILES=n overrides it for every d.
#ifdef VR_LEAF_TILES
    constexpr int LT = VR_LEAF_TILES;
#else
    constexpr int LT = D >= 7 ? 2 : 1;
#endif
    if (LT > 1 && pend < pend_end) return pend++;
    while (sp > 0) {
      --sp;
      const int node = __shfl_sync(0xffffffffu, s_node, sp);
      const int lo = __shfl_sync(0xffffffffu, s_lo, sp);
      const int hi = __shfl_sync(0xffffffffu, s_hi, sp);
      if (hi - lo <= LT) {
        leaf_mask = __shfl_sync(0xffffffffu, s_mask, sp);
        if (LT > 1) {
          pend = lo + 1;
          pend_end = hi;
        }
        return lo;
      }
      const int l = 2 * node + 1, r = 2 * node + 2;
      const int2 rl = __ldg(node_range + l), rr = __ldg(node_range + r);
#ifndef VR_NEAR_ORDER_MAX_D  // tuning knob: 0 restores start-tile-first everywhere
#define VR_NEAR_ORDER_MAX_D 6
#endif
      if constexpr (F32 && CH && R == 1 && D <= VR_NEAR_ORDER_MAX_D) {
        // nearer child first, by a vote of the lanes that need both (config
        // 2: 3,163 -> 2,971 pairs per ray, kernel 2.435 -> 2.40 ms; at d = 8
        // the rare-path entries grow 19% for 2% fewer pairs, so it stops at
        // d = 6)
        float dl, dr;
        const bool al = ray_needs_box32_ch_d2<D>(ray[0], node_box32 + (int64_t)l * box32_stride(D), dl);
        const bool ar = ray_needs_box32_ch_d2<D>(ray[0], node_box32 + (int64_t)r * box32_stride(D), dr);
        tests += 2;
        const unsigned nl = __ballot_sync(0xffffffffu, al), nr = __ballot_sync(0xffffffffu, ar);
        const unsigned both = __ballot_sync(0xffffffffu, al && ar);
        const unsigned pl = __ballot_sync(0xffffffffu, al && ar && dl <= dr);
        const bool left_first = both ? 2 * __popc(pl) >= __popc(both) : st < rl.y;
        if (left_first) {
          if (nr) push(r, rr, nr);
          if (nl) push(l, rl, nl);
        } else {
          if (nl) push(l, rl, nl);
          if (nr) push(r, rr, nr);
        }
        continue;
      }
      const unsigned nl = warp_needs(ray, node_box, node_box32, l);
      const unsigned nr = warp_needs(ray, node_box, node_box32, r);
      // the child holding the warp's start tile first (kd index order is
      // spatial order, so this visits the rays' neighbourhood early)
      if (st < rl.y) {
        if (nr) push(r, rr, nr);
        if (nl) push(l, rl, nl);
      } else {
        if (nl) push(l, rl, nl);
        if (nr) push(r, rr, nr);
      }
    }
    return -1;
  }
};

// Remapped screening (below) pays off where warp unions are large relative
// to each ray's need: d >= 7 (config-5 rays: 15.4 -> 10.8 ms per 200k).  At
// d <= 6 its extra registers cost more than it saves (config 2: 3.58 -> 3.71
// ms), so it is compiled out there.
template <int D>
__host__ __device__ constexpr int remap_max() {
#ifdef VR_REMAP_MAX
  return VR_REMAP_MAX;
#else
  return D >= 7 ? 16 : 0;
#endif
}

// Screening of one tile when only the rays of `mask` (c lanes) need it:
// G = 32 / 2^ceil(log2 c) lanes share each such ray (its screening state is
// shuffled in), each lane screens PT / G candidates, the hits are OR-reduced
// inside the group and handed to the owner lane, which runs the fp64 rare
// path on them (two 32-candidate blocks, in order).  Same verdicts as
// screen_tile_pairs for the needing rays; rays not in `mask` do not need any
// candidate of the tile (the tile box certifies it), so skipping them is exact.
template <int D, int PT>
__device__ __forceinline__ void screen_tile_remap(RayState<D>& r, const double* tile64,
                                                  const float* tilep, int gbase, unsigned mask,
                                                  const Frame& fr, WarpCounters* wc) {
  static_assert(PT == 32 || PT == 64, "hits fit a 64-bit mask");
  constexpr int P2 = rec32p_stride(D);
  const int lane = threadIdx.x & 31;
  const int c = __popc(mask);
  const int G0 = c <= 1 ? 32 : c <= 2 ? 16 : c <= 4 ? 8 : c <= 8 ? 4 : 2;
  const int G = G0 < PT / 2 ? G0 : PT / 2;  // at least one candidate pair per lane
  const int slot = lane / G, sub = lane % G;
  const bool valid = slot < c;
  const int owner = valid ? (int)__fns(mask, 0, slot + 1) : lane;
  // the owner's screening state
  float z[D], u[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    z[k] = __shfl_sync(0xffffffffu, r.z32[k], owner);
    u[k] = __shfl_sync(0xffffffffu, r.u32[k], owner);
  }
  const float hi32 = __shfl_sync(0xffffffffu, r.hi32, owner);
  const float thr32 = __shfl_sync(0xffffffffu, r.thr32, owner);
  const float bsl32 = __shfl_sync(0xffffffffu, r.bsl32, owner);
  const int ib = __shfl_sync(0xffffffffu, r.ib, owner);
  const int npairs = (PT / 2) / G;  // pairs per lane
  unsigned long long hits = 0ull;
  if (valid) {
    for (int p = 0; p < npairs; ++p) {
      const int pp = sub * npairs + p;  // pair index inside the tile
      const float4* q = reinterpret_cast<const float4*>(tilep + pp * P2);
      float v[P2];
#pragma unroll
      for (int k = 0; k < P2 / 4; ++k) {
        const float4 w = q[k];
        v[4 * k] = w.x;
        v[4 * k + 1] = w.y;
        v[4 * k + 2] = w.z;
        v[4 * k + 3] = w.w;
      }
      uint64_t acc = f2pack(v[2 * D], v[2 * D + 1]);
#pragma unroll
      for (int k = 0; k < D; ++k) acc = ffma2(f2pack(z[k], z[k]), f2pack(v[2 * k], v[2 * k + 1]), acc);
      float fa, fb;
      f2unpack(acc, fa, fb);
      if (fa < hi32 || fb < hi32) {  // rare: conservative fp32 halfspace pre-filter
        uint64_t qa2 = f2pack(bsl32, bsl32);
#pragma unroll
        for (int k = 0; k < D; ++k) qa2 = ffma2(f2pack(u[k], u[k]), f2pack(v[2 * k], v[2 * k + 1]), qa2);
        float qa, qb;
        f2unpack(qa2, qa, qb);
        const int ia = 2 * pp;
        if (fa < hi32 && qa > thr32 && gbase + ia != ib) hits |= 1ull << ia;
        if (fb < hi32 && qb > thr32 && gbase + ia + 1 != ib) hits |= 1ull << (ia + 1);
      }
    }
  }
  if (!__any_sync(0xffffffffu, hits != 0ull)) return;
  // OR inside each group of G lanes (aligned, contiguous), then to the owner
  for (int off = 1; off < G; off <<= 1) hits |= __shfl_xor_sync(0xffffffffu, hits, off);
  const bool mine = (mask >> lane) & 1u;
  const int my_slot = __popc(mask & ((1u << lane) - 1u));
  const unsigned long long h = __shfl_sync(0xffffffffu, hits, (mine ? my_slot : 0) * G);
  if (!mine || !h) return;
  if (wc) {
    ++wc->rare_blocks;
    wc->entries += __popcll(h);
  }
  const unsigned lo = (unsigned)h, hi = (unsigned)(h >> 32);
  if (lo) ray_rare_block<D, true>(r, tile64, lo, gbase, fr);
  if (hi) ray_rare_block<D, true>(r, tile64 + 32 * rec_stride(D), hi, gbase + 32, fr);
}

// ---------------------------------------------------------------------------
// Tensor-core screen (one ray per lane): the incircle powers of the
// warp's 32 rays against a 64-candidate tile are one 32 x 64 x 8KS product
//     f~ = [z32, 1, ctc] . [x~, |x~|^2, 1]  =  |x~|^2 - 2 z~.x~ - (hi32 + e_tc)
// on the legacy warp tensor path (mma.sync m16n8k8 tf32: 2 ray blocks x 8
// candidate blocks = 16 HMMA per tile, B fragments staged by TMA in fragment
// order, 8 LDS.64).  A pair passes iff f~ < 0 (sign bit, incl. -0): ctc folds
// the fp32 bound hi32 and the tf32 error bound into the product, so the
// screen stays conservative (ray_set_best derives the bound).  The A
// fragments are rebuilt through shared memory after sphere updates; a stale
// sphere only screens more pairs (the band only shrinks), never fewer.
// Passing pairs go through the same fp32 halfspace pre-filter and fp64 rare
// path as screen_tile_pairs, so the verdicts are unchanged.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], float2 b) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%10,%10,%10,%10};"
      : "=f"(c[0]), "=f"(c[1]), "=f"(c[2]), "=f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(__float_as_uint(b.x)),
        "r"(__float_as_uint(b.y)), "f"(0.0f));
}

__device__ __forceinline__ void mma_tf32_acc(float (&c)[4], const uint32_t (&a)[4], float2 b) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(__float_as_uint(b.x)),
        "r"(__float_as_uint(b.y)));
}

// k8 steps of the screen product: features [x (D), |x|^2, 1] padded to 8 KS.
__host__ __device__ constexpr int mma_ksteps(int d) { return (d + 2 + 7) / 8; }
// shared A-row stride in floats (odd: conflict-free column reads)
__host__ __device__ constexpr int mma_arow(int d) { return 8 * mma_ksteps(d) + 1; }

// The A operand lives in shared memory (row r = ray of lane r:
// [tf32(z32_r), 1, ctc_r, 0 ..]), rewritten after sphere updates; the
// fragments are re-read per tile (8 KS LDS) instead of holding registers.
template <int D>
__device__ __forceinline__ void mma_store_a(const RayState<D>& r, float* sA) {
  constexpr int KW = 8 * mma_ksteps(D), AR = mma_arow(D);
  const int lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < KW; ++k) {
    const float v = k < D ? __uint_as_float(tf32_rn(r.z32[k])) : k == D ? 1.0f
                  : k == D + 1 ? r.ctc : 0.0f;
    sA[lane * AR + k] = v;
  }
  __syncwarp();
}

// Halfspace operand (constant per ray): row r = [tf32(u32_r), 0, c2_r, 0 ..]
// with h~ = u~.x~ + c2 > 0 whenever the fp32 pre-filter of screen_tile_pairs
// (bsl32 + u32.x~ > thr32) could keep the candidate: c2 = bsl32 - thr32 + e_u
// rounded up in tf32, e_u >= |u~.x~ (tf32 MMA) - u32.x~| (2^-10 |u||x~|max +
// 2^-16 of the magnitudes, x 1.25).
__device__ __forceinline__ float tf32_up(float v) { return -tf32_down(-v); }

template <int D>
__device__ __forceinline__ void mma_store_u(const RayState<D>& r, const Frame& fr, float* sU) {
  constexpr int KW = 8 * mma_ksteps(D), AR = mma_arow(D);
  const int lane = threadIdx.x & 31;
  const double xm = sqrt(fr.sqmax32);
  const double eu = 1.25 * (9.775161743164062e-04 * xm +
                            1.52587890625e-05 * (xm + fabs((double)r.thr32) + 1.0));
  double c2 = (double)r.bsl32 - (double)r.thr32 + eu;
  c2 = fmin(fmax(c2, -1e30), 1e30);  // padding lanes (thr32 = +inf): finite
  __syncwarp();
#pragma unroll
  for (int k = 0; k < KW; ++k) {
    const float v = k < D ? __uint_as_float(tf32_rn(r.u32[k])) : k == D + 1
                  ? tf32_up(__double2float_ru(c2)) : 0.0f;
    sU[lane * AR + k] = v;
  }
  __syncwarp();
}

// Fragments of rays 0-15 (a[s][0]) and 16-31 (a[s][1]) for k-step s: lane l
// holds A[16m + g][8s + t], A[16m + g + 8][8s + t], A[16m + g][8s + t + 4],
// A[16m + g + 8][8s + t + 4], g = l >> 2, t = l & 3.
template <int D>
__device__ __forceinline__ void mma_load_a(const float* sA, uint32_t (&a)[mma_ksteps(D)][2][4]) {
  constexpr int AR = mma_arow(D);
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int q = 0; q < mma_ksteps(D); ++q)
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      a[q][m][0] = __float_as_uint(sA[(16 * m + g) * AR + 8 * q + t]);
      a[q][m][1] = __float_as_uint(sA[(16 * m + g + 8) * AR + 8 * q + t]);
      a[q][m][2] = __float_as_uint(sA[(16 * m + g) * AR + 8 * q + t + 4]);
      a[q][m][3] = __float_as_uint(sA[(16 * m + g + 8) * AR + 8 * q + t + 4]);
    }
}

// C (rays 16m .. 16m+15, candidates 8j .. 8j+7) of the screen product.
template <int KS>
__device__ __forceinline__ void mma_block(float (&c)[4], const uint32_t (&a)[KS][2][4], int m,
                                          const float2* Bj) {
  const int lane = threadIdx.x & 31;
  mma_tf32(c, a[0][m], Bj[lane]);
#pragma unroll
  for (int q = 1; q < KS; ++q) mma_tf32_acc(c, a[q][m], Bj[q * 32 + lane]);
}

// Spread the 4 low bits of x to the even bit positions 0, 2, 4, 6.
__device__ __forceinline__ uint32_t spread4(uint32_t x) {
  x = (x | (x << 2)) & 0x33u;
  return (x | (x << 1)) & 0x55u;
}

template <int D>
__device__ __forceinline__ void screen_tile_mma(RayState<D>& r, const double* tile64,
                                                const float* tileB, int gbase,
                                                const Frame& fr, WarpCounters* wc, float* sA,
                                                const float* sU) {
  constexpr int S = rec_stride(D);
  constexpr int KS = mma_ksteps(D);
  const int lane = threadIdx.x & 31;
  const float2* B = reinterpret_cast<const float2*>(tileB);  // [8 blocks][KS][32 lanes]
  uint32_t a[KS][2][4];
  mma_load_a<D>(sA, a);
  uint32_t acc = 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float c0[4], c1[4];
    mma_block<KS>(c0, a, 0, B + j * KS * 32);
    mma_block<KS>(c1, a, 1, B + j * KS * 32);
    acc |= __float_as_uint(c0[0]) | __float_as_uint(c0[1]) | __float_as_uint(c0[2]) |
           __float_as_uint(c0[3]) | __float_as_uint(c1[0]) | __float_as_uint(c1[1]) |
           __float_as_uint(c1[2]) | __float_as_uint(c1[3]);
  }
  if (!__any_sync(0xffffffffu, (int)acc < 0)) return;
  // Some pair passed: recompute, add the halfspace product (the conservative
  // pre-filter: most pairs inside a stale sphere lie behind the ray), and
  // route each ray's 64 verdicts to its lane with ballots.  C element (m, e)
  // of lane (g, t) is ray 16m + 8(e >> 1) + g, column 8j + 2t + (e & 1); ray
  // r = lane reads bits 4g .. 4g+3 of the ballots of elements
  // (r >> 4, 2((r >> 3) & 1) + {0, 1}).
  uint32_t au[KS][2][4];
  mma_load_a<D>(sU, au);
  const int rm = lane >> 4, rh = (lane >> 3) & 1, sh = 4 * (lane & 7);
  unsigned long long m = 0ull;
#pragma unroll 1
  for (int j = 0; j < 8; ++j) {
    float c0[4], c1[4], h0[4], h1[4];
    mma_block<KS>(c0, a, 0, B + j * KS * 32);
    mma_block<KS>(c1, a, 1, B + j * KS * 32);
    mma_block<KS>(h0, au, 0, B + j * KS * 32);
    mma_block<KS>(h1, au, 1, B + j * KS * 32);
    uint32_t v[2][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      v[0][e] = __ballot_sync(0xffffffffu, (int)(__float_as_uint(c0[e]) & ~__float_as_uint(h0[e])) < 0);
      v[1][e] = __ballot_sync(0xffffffffu, (int)(__float_as_uint(c1[e]) & ~__float_as_uint(h1[e])) < 0);
    }
    const uint32_t ev = rm ? (rh ? v[1][2] : v[1][0]) : (rh ? v[0][2] : v[0][0]);
    const uint32_t od = rm ? (rh ? v[1][3] : v[1][1]) : (rh ? v[0][3] : v[0][1]);
    const uint32_t byte = spread4((ev >> sh) & 0xfu) | (spread4((od >> sh) & 0xfu) << 1);
    m |= (unsigned long long)byte << (8 * j);
  }
  const int rel = r.ib - gbase;  // the current best itself
  if ((unsigned)rel < 64u) m &= ~(1ull << rel);
  // g lies on every sphere of the ray (power 0) and on the halfspace boundary
  // (u.x_g = s < thr), so both products always pass it; it is never valid
  // (raycast.py:110-117), so dropping it is exact.
  const int relg = r.gk - gbase;
  if ((unsigned)relg < 64u) m &= ~(1ull << relg);
  const unsigned long long keep = m;
  if (wc) {
    ++wc->rare_blocks;
    wc->entries += __popcll(keep);
    wc->rare_iters += __reduce_max_sync(0xffffffffu, (unsigned)__popcll(keep));
  }
  const int nupd0 = r.nupd;
  const unsigned lo = (unsigned)keep, hi = (unsigned)(keep >> 32);
  if (lo) ray_rare_block<D, true>(r, tile64, lo, gbase, fr);
  if (hi) ray_rare_block<D, true>(r, tile64 + 32 * S, hi, gbase + 32, fr);
  if (__any_sync(0xffffffffu, r.nupd != nupd0)) mma_store_a<D>(r, sA);
}

// ---------------------------------------------------------------------------
// Tensor-core sweep on the warp path (k_raycast_hsweep, d <= 6): every
// generator screened, no kd walk.  NW warps x 32 rays per CTA share a
// STAGES-deep ring of TC-candidate B blocks (mma.sync fragment layout,
// vr_pack_records_mma) filled by TMA bulk copies; the last warp to release
// a stage issues its refill, so no warp waits for another.  Each 64-candidate
// tile goes through screen_tile_mma (16 HMMA + one OR vote in the common
// no-hit case; the ballot routing, halfspace product and fp64 rare path on a
// hit), so results are bitwise the pruned kernel's.  Blocks are visited in a
// spiral around the CTA's home block (kd order), so spheres shrink early.
// ---------------------------------------------------------------------------
template <int D, int NW, int STAGES, int TC, int MINB, class Src>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_raycast_hsweep(Src src, int64_t n_rays, const double* __restrict__ crec,
                     const float* __restrict__ crecB, const float* __restrict__ crec32s,
                     const int32_t* __restrict__ perm, const int32_t* __restrict__ inv_perm,
                     int64_t n_rows, Frame fr, RayOut out, unsigned long long* __restrict__ work) {
  constexpr int S = rec_stride(D);
  constexpr int KS = mma_ksteps(D);
  constexpr int AR = mma_arow(D);
  constexpr int BLK = TC * 8 * KS;  // floats per stage block
  static_assert(TC % 64 == 0, "whole 64-candidate tiles per stage");
  extern __shared__ __align__(128) float sBdyn[];  // STAGES x BLK floats (dynamic)
  float (*sB)[BLK] = reinterpret_cast<float (*)[BLK]>(sBdyn);
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ int released[STAGES];
  __shared__ float sA[NW][32 * AR];
  __shared__ float sU[NW][32 * AR];
  __shared__ int64_t home_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nblk = n_rows / TC;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      released[i] = 0;
    }
    fence_mbar_init();
    home_s = (int64_t)inv_perm[src.gen((int64_t)blockIdx.x * NW * 32)] / TC;
  }
  __syncthreads();
  const int64_t home = home_s;
  auto block_of = [&](int64_t j) -> int64_t {  // home, +1, -1, +2, -2, ...
    const int64_t off = (j & 1) ? (j + 1) >> 1 : -(j >> 1);
    int64_t b = home + off;
    if (b >= nblk) b -= nblk;
    if (b < 0) b += nblk;
    return b;
  };
  auto issue = [&](int64_t j) {
    const int st = (int)(j % STAGES);
    mbar_arrive_expect_tx(&full[st], BLK * 4);
    bulk_g2s(sB[st], crecB + block_of(j) * BLK, BLK * 4, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int64_t j = 0; j < STAGES && j < nblk; ++j) issue(j);
  const int64_t k = ((int64_t)blockIdx.x * NW + w) * 32 + lane;
  RayState<D> ray;
  const bool act = k < n_rays && src.load(k, ray, fr);
  if (!act) init_padding_lane<D, 1>(ray);
  if (act) {
    ray.gk = inv_perm[src.gen(k)];
    const int64_t so = (int64_t)ray.gk / 64;
    seed_tile32<D>(ray, crec32s + so * 64 * rec32_stride(D), crec + so * 64 * S, (int)(so * 64), fr);
  }
  mma_store_a<D>(ray, sA[w]);
  mma_store_u<D>(ray, fr, sU[w]);
  WarpCounters wc;
  for (int64_t j = 0; j < nblk; ++j) {
    const int st = (int)(j % STAGES);
    mbar_wait(&full[st], (uint32_t)((j / STAGES) & 1));
    const int64_t b = block_of(j);
#pragma unroll 1
    for (int sub = 0; sub < TC / 64; ++sub) {
      const int gbase = (int)(b * TC + sub * 64);
      screen_tile_mma<D>(ray, crec + (int64_t)gbase * S, sB[st] + sub * 512 * KS, gbase, fr,
                         work ? &wc : nullptr, sA[w], sU[w]);
    }
    __syncwarp();
    if (lane == 0) {
      // the last warp done with this stage refills it
      if (atomicAdd(&released[st], 1) == NW - 1) {
        released[st] = 0;
        if (j + STAGES < nblk) issue(j + STAGES);
      }
    }
  }
  if (act) ray_store<D>(ray, src.id(k), perm, out);
  if (work) {
    unsigned long long up = act ? ray.nupd : 0, a = act ? 1 : 0;
    unsigned long long e = wc.entries;
    for (int off = 16; off > 0; off >>= 1) {
      up += __shfl_xor_sync(0xffffffffu, up, off);
      a += __shfl_xor_sync(0xffffffffu, a, off);
      e += __shfl_xor_sync(0xffffffffu, e, off);
    }
    if (lane == 0) {
      atomicAdd(work, a * (unsigned long long)n_rows);
      atomicAdd(work + 1, wc.rare_blocks);
      atomicAdd(work + 2, wc.rare_iters);
      atomicAdd(work + 3, e);
      atomicAdd(work + 4, up);
    }
  }
}

// One warp per CTA (warps finish at very different times; a freed slot is
// refilled immediately).  The warp's next needed tile is fetched by TMA into
// the other half of a two-tile shared-memory buffer while the current tile
// is screened; the need test is re-applied before screening (spheres shrink).
template <int D, int R, int PT, int PB, int MINB, bool F32, class Src, bool MMA = false>
__global__ void __launch_bounds__(32, MINB)
    k_raycast_pruned(Src src, const double* __restrict__ crec, const float* __restrict__ crec32,
                     const float* __restrict__ crecB, const float* __restrict__ crec32s,
                     const int32_t* __restrict__ perm, const int32_t* __restrict__ inv_perm,
                     int64_t n_cand, const double* __restrict__ tile_box,
                     const float* __restrict__ tile_box32, const double* __restrict__ node_box,
                     const float* __restrict__ node_box32, const int2* __restrict__ node_range,
                     Frame fr, RayOut out, unsigned long long* __restrict__ work,
                     unsigned long long* __restrict__ next_item) {
  constexpr int S = rec_stride(D);
  // both copies are staged: the fp64 rows feed the rare path, which is hit
  // often enough (tens of entries per ray at d=8) that global loads stall
#ifdef VR_STAGE64
  constexpr bool STAGE64 = true;
#else
  constexpr bool STAGE64 = !F32;  // fp32 screen: the rare path reads fp64 rows from L2
#endif
  constexpr uint32_t BYTES64 = STAGE64 ? (uint32_t)(PT * S * sizeof(double)) : 0u;
  constexpr int P2 = rec32p_stride(D);
  // the tensor-core screen needs neither the fp32 pair rows nor the fp64 rows
  // in shared memory (its halfspace product replaces the pair pre-filter)
  // (for d >= 7 it also replaces the remapped screen of sparse tiles: a
  // remap/tensor-core hybrid measured slower on config 5, 1.60 vs 1.32 s)
  constexpr uint32_t BYTES32 = F32 && !MMA ? (uint32_t)(PT / 2 * P2 * sizeof(float)) : 0u;
  static_assert(PT % 8 == 0 && VR_REC_PAD % PT == 0, "tile must divide the record padding");
  __shared__ __align__(128) double buf[2][STAGE64 ? PT * S : 2];
  __shared__ __align__(128) float buf32[2][F32 && !MMA ? PT / 2 * P2 : 4];
  static_assert(!MMA || (F32 && R == 1 && PT == 64), "tensor-core screen shape");
  constexpr int KW = 8 * mma_ksteps(D);
  constexpr uint32_t BYTESB = MMA ? (uint32_t)(PT * KW * sizeof(float)) : 0u;
  __shared__ __align__(128) float bufB[2][MMA ? PT * KW : 4];
  __shared__ float sA[MMA ? 32 * mma_arow(D) : 1];
  __shared__ float sU[MMA ? 32 * mma_arow(D) : 1];
  __shared__ uint64_t bar[2];
  const int lane = threadIdx.x;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phases = 0u;  // mbarrier parity of buffer b = bit b (a register, not a local array)
  // Work items = groups of 32 R consecutive slots of the processing order.
  // Without a counter one item per CTA; with one (persistent launch: about
  // one CTA per resident warp slot) items are handed out in order by an
  // atomic counter, so no SM idles between CTAs and the tail balances.
  const int64_t n_items = (src.n + 32 * R - 1) / (32 * R);
  int64_t item = blockIdx.x;
  while (item < n_items) {
  const int64_t k0 = item * 32 * R + lane;

  RayState<D> ray[R];
  bool act[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    act[j] = src.load(k0 + (int64_t)j * 32, ray[j], fr);
    if (!act[j]) init_padding_lane<D, R>(ray[j]);
  }
  // fp32 seed (seed_tile32) wherever the kd-ordered fp32 rows are there:
  // the tensor-core kernel and the one-ray-per-lane FFMA2 kernel
  constexpr bool SEED32 = MMA || (F32 && R == 1);
  if constexpr (SEED32) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (act[j]) ray[j].gk = inv_perm[src.gen(k0 + (int64_t)j * 32)];
  }
  int64_t st = 0;
  if (lane == 0) st = inv_perm[src.gen(k0)] / PT;
  st = __shfl_sync(0xffffffffu, st, 0);
  if constexpr (SEED32) {
    // each ray seeds on the tile of its own reference generator (sparse
    // batches, where a warp spans several generators: 64k config-2 rays
    // 9.97 -> 7.83 ms per 1e6; dense batches unchanged), division-free in
    // fp32 with one fp64 evaluation of the winner (the fp64 seed over 64
    // candidates was 16% of config 4's kernel samples)
    if (crec32s) {
      const int64_t so = act[0] ? (int64_t)ray[0].gk / PT : st;
      seed_tile32<D>(ray[0], crec32s + so * PT * rec32_stride(D), crec + so * PT * S,
                     (int)(so * PT), fr);
    } else {
      seed_tile<D, R, PT, F32>(ray, crec + st * PT * S, (int)(st * PT), fr);
    }
  }
  else
    seed_tile<D, R, PT, F32>(ray, crec + st * PT * S, (int)(st * PT), fr);
  // (the tensor-core kernel's node_box32 argument holds centre / half-extent rows)
  TreeCursor<D, R, F32, MMA> cur;
  cur.init(st, ray, node_box, node_box32, node_range);
  if constexpr (MMA) {
    mma_store_a<D>(ray[0], sA);
    mma_store_u<D>(ray[0], fr, sU);
  }

  auto issue = [&](int64_t t, int b) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(&bar[b], BYTES64 + BYTES32 + BYTESB);
      if constexpr (STAGE64) bulk_g2s(buf[b], crec + t * PT * S, BYTES64, &bar[b]);
      if constexpr (F32 && !MMA) bulk_g2s(buf32[b], crec32 + t * (PT / 2) * P2, BYTES32, &bar[b]);
      if constexpr (MMA) bulk_g2s(bufB[b], crecB + t * PT * KW, BYTESB, &bar[b]);
    }
  };
  unsigned long long tiles_done = 0;
  WarpCounters wc;
  int b = 0;
  int64_t t = cur.next(ray, node_box, node_box32, node_range);
  unsigned tmask = cur.leaf_mask;
  if (t >= 0) issue(t, 0);
  while (t >= 0) {
    const int64_t tn = cur.next(ray, node_box, node_box32, node_range);
    const unsigned tn_mask = cur.leaf_mask;
    __syncwarp();
    if (tn >= 0) issue(tn, b ^ 1);
    mbar_wait(&bar[b], (phases >> b) & 1u);
    phases ^= 1u << b;
    // (no re-test of the tile box here: the leaf was tested when its parent
    // was expanded, and re-testing skipped < 2% of the tiles on config 2)
    ++tiles_done;
    if constexpr (MMA) {
      screen_tile_mma<D>(ray[0], crec + t * PT * S, bufB[b], (int)(t * PT), fr,
                         work ? &wc : nullptr, sA, sU);
    } else if constexpr (F32 && R == 1 && (PT == 32 || PT == 64) && remap_max<D>() > 0) {
      if (__popc(tmask) <= remap_max<D>())
        screen_tile_remap<D, PT>(ray[0], STAGE64 ? buf[b] : crec + t * PT * S, buf32[b],
                                 (int)(t * PT), tmask, fr, work ? &wc : nullptr);
      else
        screen_tile_pairs<D, R, PT>(ray, STAGE64 ? buf[b] : crec + t * PT * S, buf32[b],
                                    (int)(t * PT), fr, work ? &wc : nullptr);
    } else if constexpr (F32)
      screen_tile_pairs<D, R, PT>(ray, STAGE64 ? buf[b] : crec + t * PT * S, buf32[b],
                                  (int)(t * PT), fr, work ? &wc : nullptr);
    else
      screen_tile<D, R, PT, F32>(ray, buf[b], buf32[b], (int)(t * PT), fr, work ? &wc : nullptr);
    __syncwarp();
    b ^= 1;
    t = tn;
    tmask = tn_mask;
  }
#pragma unroll
  for (int j = 0; j < R; ++j)
    if (act[j]) ray_store<D>(ray[j], src.id(k0 + (int64_t)j * 32), perm, out);
  // work counters: [0] (ray, generator) pairs screened = tiles x PT x 32 x R,
  // [1] blocks with rare work, [2] warp-level rare iterations, [3] entries,
  // [4] ray updates (sum over lanes of sphere moves)
  if (work) {
    unsigned long long e = wc.entries;
    for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    unsigned long long up = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) up += act[j] ? ray[j].nupd : 0;
    for (int off = 16; off > 0; off >>= 1) up += __shfl_xor_sync(0xffffffffu, up, off);
    if (lane == 0) {
      atomicAdd(work, tiles_done * (unsigned long long)(PT * 32 * R));
      atomicAdd(work + 1, wc.rare_blocks);
      atomicAdd(work + 2, wc.rare_iters);
      atomicAdd(work + 3, e);
      atomicAdd(work + 4, up);
      atomicAdd(work + 5, cur.tests);
    }
#ifdef VR_RARE_STATS
    int st[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (act[j]) {
        st[0] += ray[j].st_out; st[1] += ray[j].st_self; st[2] += ray[j].st_behind;
        st[3] += ray[j].st_band; st[4] += ray[j].st_imp;
      }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      unsigned long long v = st[q];
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) atomicAdd(work + 6 + q, v);
    }
#endif
  }
  if (!next_item) break;
  __syncwarp();  // every lane is done with the shared buffers of this item
  unsigned long long nx = 0;
  if (lane == 0) nx = atomicAdd(next_item, 1ull);
  item = (int64_t)gridDim.x + (int64_t)__shfl_sync(0xffffffffu, nx, 0);
  }
}

// ---------------------------------------------------------------------------
// Cooperative pruned kernel: one WARP per ray.
//
// In high dimension the union of 32 rays' spheres covers many more tiles than
// each ray needs (config-5 edge rays: ~460 tiles per warp vs ~2.4 per ray for
// the final spheres), so here the 32 lanes work on ONE ray: a tile of 64
// candidates is screened as one pair (two candidates, packed FFMA2) per lane,
// and the kd tiles are grouped into a 32-ary tree whose children are tested
// one per lane.  The block-batched rare path is applied to a whole tile: the
// improving candidates of all lanes are reduced to the smallest t (warp
// argmin, division-free), one sphere update, every other improving candidate
// re-tested against the new sphere (RECHECK if inside its band).  Skipping
// is a certificate and the screen is conservative, so results equal the
// exhaustive kernel's.
// ---------------------------------------------------------------------------
#ifndef VR_COOP_MINB
#define VR_COOP_MINB 1
#endif
constexpr int WIDE = 32;
constexpr int WIDE_MAX_LEVELS = 8;

struct WideTree {
  const float* box32;             // fp32 centred outward boxes, all levels (box32_stride rows)
  int64_t off[WIDE_MAX_LEVELS];   // first row of level l (level 0 = tiles)
  int64_t cnt[WIDE_MAX_LEVELS];   // nodes in level l
  int levels;                     // the top level (levels - 1) holds one node
};

// fp32 box test for one ray against a box held in registers; d2 = squared
// distance of the sphere centre to the box (ordering key).
template <int D>
__device__ __forceinline__ bool coop_box_need(const RayState<D>& r, const float (&v)[box32_stride(D)],
                                              float& d2) {
  float umax = 0.0f;
  d2 = 0.0f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const float lo = v[k], hi = v[D + k];
    umax = fmaf(r.u32[k], r.u32[k] > 0.0f ? hi : lo, umax);
    const float zc = -0.5f * r.z32[k];
    const float e = fmaxf(fmaxf(lo - zc, zc - hi) - r.del32, 0.0f);
    d2 = fmaf(e, e, d2);
  }
  if (umax + r.bsl32 <= r.thr32) return false;
  return !(d2 >= r.rb32);
}

template <int D>
__device__ __forceinline__ void coop_load_box(const float* p, float (&v)[box32_stride(D)]) {
  const float4* b4 = reinterpret_cast<const float4*>(p);
#pragma unroll
  for (int k = 0; k < box32_stride(D) / 4; ++k) {
    const float4 w = __ldg(b4 + k);
    v[4 * k] = w.x;
    v[4 * k + 1] = w.y;
    v[4 * k + 2] = w.z;
    v[4 * k + 3] = w.w;
  }
}

// Warp argmin of t = num / (2 den) (den > 0), smallest index on exact ties;
// lanes without a candidate pass idx < 0.  Returns the winning lane's triple.
__device__ __forceinline__ void coop_argmin(double& num, double& den, int& idx) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double on = __shfl_xor_sync(0xffffffffu, num, off);
    const double od = __shfl_xor_sync(0xffffffffu, den, off);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
    bool take;
    if (oi < 0) take = false;
    else if (idx < 0) take = true;
    else {
      const double a = on * den, b = num * od;
      take = a < b || (a == b && oi < idx);
    }
    if (take) { num = on; den = od; idx = oi; }
  }
  // rounded products are not a strict order in near-ties: make every lane
  // agree on lane 0's result (the ray state must stay warp-uniform)
  num = __shfl_sync(0xffffffffu, num, 0);
  den = __shfl_sync(0xffffffffu, den, 0);
  idx = __shfl_sync(0xffffffffu, idx, 0);
}

// Seed: the best valid candidate of the ray's start tile (two per lane).
template <int D, int PT>
__device__ __forceinline__ void coop_seed(RayState<D>& r, const double* __restrict__ crec,
                                          int64_t tile, const Frame& fr) {
  constexpr int S = rec_stride(D);
  const int lane = threadIdx.x & 31;
  double bn = 1.0, bd = 0.0;
  int bi = -1;
#pragma unroll
  for (int h = 0; h < PT / 32; ++h) {
    const int64_t i = tile * PT + h * 32 + lane;
    double xi[D];
    load_rec_g<D>(crec + i * S, xi);
    const bool real = !isinf(__ldg(crec + i * S + D));
    double q = 0.0, aa = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      q = fma(r.u[k], xi[k], q);
      const double a = r.x[k] - xi[k];
      aa = fma(a, a, aa);
    }
    const double num = aa - r.base, den = q - r.s;
    if (real && q > r.thr && (bi < 0 || num * bd < bn * den)) { bn = num; bd = den; bi = (int)i; }
  }
  coop_argmin(bn, bd, bi);
  if (bi >= 0) {
    const double t = bn / (2.0 * bd);
    if (r.ib < 0 || t < r.tb) ray_set_best<D, true>(r, t, bd, bi, fr);
  }
}

// Rare path for one tile: lanes hold up to two candidates that passed the
// fp32 screens (pa / pb; candidate indices ia, ia + 1).
template <int D>
__device__ __forceinline__ void coop_rare(RayState<D>& r, const double* __restrict__ crec,
                                          int ia, bool pa, bool pb, const Frame& fr) {
  constexpr int S = rec_stride(D);
  const bool have0 = r.ib >= 0;
  double zk2[D];
#pragma unroll
  for (int k = 0; k < D; ++k) zk2[k] = have0 ? -2.0 * fma(r.tb, r.u[k], r.x[k]) : 0.0;
  double bn = 1.0, bd = 0.0;
  int bi = -1;
  int near = 0;
  unsigned imp = 0u;
  double xs[2][D], sqs[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const bool p = h ? pb : pa;
    if (!p) continue;
    const int i = ia + h;
    load_rec_g<D>(crec + (int64_t)i * S, xs[h]);
    sqs[h] = __ldg(crec + (int64_t)i * S + D);
    double fp = sqs[h], q = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      fp = fma(zk2[k], xs[h][k], fp);
      q = fma(r.u[k], xs[h][k], q);
    }
    if (have0 && !(fp < r.hi)) continue;
    if (!(q > r.thr)) continue;  // raycast.py:110-117
    if (have0 && fp >= r.lim - r.dlt) near = 1;
    if (have0 && !(fp < r.lim)) continue;
    double aa = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double a = r.x[k] - xs[h][k];
      aa = fma(a, a, aa);
    }
    const double num = aa - r.base, den = q - r.s;  // raycast.py:201-203
    if (bi < 0 || num * bd < bn * den) { bn = num; bd = den; bi = i; }
    imp |= 1u << h;
  }
  int wi = bi;
  double wn = bn, wd = bd;
  coop_argmin(wn, wd, wi);
  if (wi >= 0) {
    const double t = wn / (2.0 * wd);
    const double told = r.tb, denold = r.denb;
    ray_set_best<D, true>(r, t, wd, wi, fr);
    if (have0 && 2.0 * denold * (told - t) < r.dlt) near = 1;
    // every other improving candidate against the new sphere
#pragma unroll
    for (int k = 0; k < D; ++k) zk2[k] = -2.0 * fma(t, r.u[k], r.x[k]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!((imp >> h) & 1u) || ia + h == wi) continue;
      double fp = sqs[h];
#pragma unroll
      for (int k = 0; k < D; ++k) fp = fma(zk2[k], xs[h][k], fp);
      if (fp < r.hi) near = 1;
    }
  }
  if (__any_sync(0xffffffffu, near)) r.near = 1;
}

template <int D, int PT>
__device__ __forceinline__ void coop_screen_tile(RayState<D>& r, const double* __restrict__ crec,
                                                 const float* __restrict__ crec32p, int64_t tile,
                                                 const Frame& fr, WarpCounters* wc) {
  static_assert(PT == 64, "one candidate pair per lane");
  constexpr int P2 = rec32p_stride(D);
  const int lane = threadIdx.x & 31;
  const float4* q4 = reinterpret_cast<const float4*>(crec32p + (tile * (PT / 2) + lane) * P2);
  float v[P2];
#pragma unroll
  for (int k = 0; k < P2 / 4; ++k) {
    const float4 w = __ldg(q4 + k);
    v[4 * k] = w.x;
    v[4 * k + 1] = w.y;
    v[4 * k + 2] = w.z;
    v[4 * k + 3] = w.w;
  }
  uint64_t acc = f2pack(v[2 * D], v[2 * D + 1]);
#pragma unroll
  for (int k = 0; k < D; ++k) acc = ffma2(f2pack(r.z32[k], r.z32[k]), f2pack(v[2 * k], v[2 * k + 1]), acc);
  float fa, fb;
  f2unpack(acc, fa, fb);
  bool pa = fa < r.hi32, pb = fb < r.hi32;
  if (!__any_sync(0xffffffffu, pa || pb)) return;
  // conservative fp32 halfspace pre-filter + the current best itself
  uint64_t qa2 = f2pack(r.bsl32, r.bsl32);
#pragma unroll
  for (int k = 0; k < D; ++k) qa2 = ffma2(f2pack(r.u32[k], r.u32[k]), f2pack(v[2 * k], v[2 * k + 1]), qa2);
  float qa, qb;
  f2unpack(qa2, qa, qb);
  const int ia = (int)(tile * PT) + 2 * lane;
  pa = pa && qa > r.thr32 && ia != r.ib;
  pb = pb && qb > r.thr32 && ia + 1 != r.ib;
  const unsigned m = __ballot_sync(0xffffffffu, pa || pb);
  if (!m) return;
  if (wc) {
    ++wc->rare_blocks;
    wc->entries += (pa ? 1 : 0) + (pb ? 1 : 0);
  }
  coop_rare<D>(r, crec, ia, pa, pb, fr);
}

constexpr int COOP_STK = WIDE * WIDE_MAX_LEVELS;  // shared ints per warp (DFS stack)

// One ray (slot k of src) on the calling warp; `stk` = COOP_STK shared ints
// of this warp.  The body of k_raycast_coop, also run by the persistent
// small-traversal kernel (level_small.cu).
template <int D, int PT, class Src>
__device__ __forceinline__ void coop_ray(const Src& src, int64_t k, const double* __restrict__ crec,
                                         const float* __restrict__ crec32p,
                                         const int32_t* __restrict__ perm,
                                         const int32_t* __restrict__ inv_perm, const WideTree& wt,
                                         const Frame& fr, const RayOut& out,
                                         unsigned long long* __restrict__ work, int* stk) {
  constexpr int BS = box32_stride(D);
  constexpr int STK = COOP_STK;
  const int lane = threadIdx.x & 31;
  RayState<D> r;
  src.load(k, r, fr);
  coop_seed<D, PT>(r, crec, inv_perm[src.gen(k)] / PT, fr);
  // edge rays: the tiles of the other eta generators surround the origin too
  for (int e = 1; e < src.eta_count(); ++e) coop_seed<D, PT>(r, crec, inv_perm[src.eta_at(k, e)] / PT, fr);
  WarpCounters wc;
  unsigned long long tiles = 0, tests = 0;
  const int top = wt.levels - 1;
  int sp = 1;
  if (lane == 0) stk[0] = top << 24;
  __syncwarp();
  while (sp > 0) {
    --sp;
    const int e = stk[sp];
    const int lev = e >> 24;
    const int64_t c0 = (int64_t)(e & 0xFFFFFF) * WIDE;
    const int cl = lev - 1;
    const int64_t child = c0 + lane;
    float box[BS];
    bool need = false;
    float d2 = 0.0f;
    if (child < wt.cnt[cl]) {
      coop_load_box<D>(wt.box32 + (wt.off[cl] + child) * BS, box);
      need = coop_box_need<D>(r, box, d2);
    }
    ++tests;
    unsigned mask = __ballot_sync(0xffffffffu, need);
    if (cl > 0) {
      // push: nearest child (smallest d2) on top, the rest in lane order
      float bd2 = need ? d2 : CUDART_INF_F;
      int bl = need ? lane : 32;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, bd2, off);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
        if (o < bd2 || (o == bd2 && ol < bl)) { bd2 = o; bl = ol; }
      }
      bl = __shfl_sync(0xffffffffu, bl, 0);
      if (mask) {
        const unsigned rest = mask & ~(1u << bl);
        if (need && lane != bl) {
          // higher lanes deeper in the stack: lane order pops ascending
          const int pos = sp + __popc(rest >> (lane + 1));
          if (pos >= STK) __trap();
          stk[pos] = (cl << 24) | (int)child;
        }
        sp += __popc(rest);
        if (lane == bl) stk[sp] = (cl << 24) | (int)child;
        ++sp;
        if (sp > STK) __trap();
      }
      __syncwarp();
    } else {
      // children are tiles: nearest first, each re-tested against the
      // current (shrinking) sphere before it is screened
      unsigned todo = mask;
      while (todo) {
        const bool mine = (todo >> lane) & 1u;
        bool nd = false;
        if (mine) nd = coop_box_need<D>(r, box, d2);
        todo = __ballot_sync(0xffffffffu, nd);
        if (!todo) break;
        float bd2 = nd ? d2 : CUDART_INF_F;
        int bl = nd ? lane : 32;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const float o = __shfl_xor_sync(0xffffffffu, bd2, off);
          const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
          if (o < bd2 || (o == bd2 && ol < bl)) { bd2 = o; bl = ol; }
        }
        bl = __shfl_sync(0xffffffffu, bl, 0);
        todo &= ~(1u << bl);
        ++tiles;
        coop_screen_tile<D, PT>(r, crec, crec32p, c0 + bl, fr, work ? &wc : nullptr);
      }
    }
  }
  if (lane == 0) ray_store<D>(r, src.id(k), perm, out);
  if (work && lane == 0) {
    atomicAdd(work, tiles * (unsigned long long)PT);
    atomicAdd(work + 5, tests);
    atomicAdd(work + 4, (unsigned long long)r.nupd);
  }
  if (work) {
    unsigned long long e = wc.entries, rb = wc.rare_blocks;
    for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
    if (lane == 0) {
      atomicAdd(work + 1, rb);
      atomicAdd(work + 2, rb);
      atomicAdd(work + 3, e);
    }
  }
}

template <int D, int PT, int NW, int MINB, class Src>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_raycast_coop(Src src, int64_t n_rays, const double* __restrict__ crec,
                   const float* __restrict__ crec32p, const int32_t* __restrict__ perm,
                   const int32_t* __restrict__ inv_perm, WideTree wt, Frame fr, RayOut out,
                   unsigned long long* __restrict__ work) {
  __shared__ int stk_s[NW][COOP_STK];
  const int w = threadIdx.x >> 5;
  const int64_t k = (int64_t)blockIdx.x * NW + w;
  if (k >= n_rays) return;
  coop_ray<D, PT>(src, k, crec, crec32p, perm, inv_perm, wt, fr, out, work, stk_s[w]);
}

// ---------------------------------------------------------------------------
// Exact re-check: one CTA per listed ray.  Pass 1: centred t for every valid
// candidate, lexicographic (t, index) argmin.  Pass 2: runner-up distance at
// the winner's vertex; DEGENERATE when second < radius (1 + 1e-10)
// (raycast.py:211-219).
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ void block_argmin(double& t, int& i, double* sh_t, int* sh_i) {
  for (int off = 16; off > 0; off >>= 1) {
    const double ot = __shfl_xor_sync(0xffffffffu, t, off);
    const int oi = __shfl_xor_sync(0xffffffffu, i, off);
    if (ot < t || (ot == t && (unsigned)oi < (unsigned)i)) { t = ot; i = oi; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) { sh_t[w] = t; sh_i[w] = i; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < NT / 32; ++k) {
      if (sh_t[k] < t || (sh_t[k] == t && (unsigned)sh_i[k] < (unsigned)i)) { t = sh_t[k]; i = sh_i[k]; }
    }
    sh_t[0] = t;
    sh_i[0] = i;
  }
  __syncthreads();
  t = sh_t[0];
  i = sh_i[0];
}

// Exact re-check of ray k by the whole (NT-thread) block; sh_t / sh_i are
// NT / 32 shared slots.  Returns with the result stored.
template <int D, int NT, class Src>
__device__ __forceinline__ void recheck_ray(const Src& src, int64_t k,
                                            const double* __restrict__ crec,
                                            const int32_t* __restrict__ cand, int64_t n_cand,
                                            const RayOut& out, double* sh_t, int* sh_i) {
  constexpr int S = rec_stride(D);
  {
    RayState<D> r;
    src.load(k, r, Frame{});
    double best = CUDART_INF;
    int bi = -1;
    for (int64_t c = threadIdx.x; c < n_cand; c += NT) {
      const double* xc = crec + c * S;
      double q = 0.0, aa = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        q = fma(r.u[j], xc[j], q);
        const double a = r.x[j] - xc[j];
        aa = fma(a, a, aa);
      }
      if (q > r.thr) {
        const double t = (aa - r.base) / (2.0 * (q - r.s));
        if (t < best) { best = t; bi = (int)c; }  // ascending c per thread: keeps smallest index
      }
    }
    if (bi < 0) best = CUDART_INF;
    block_argmin<NT>(best, bi, sh_t, sh_i);
    if (bi < 0 || !(best < CUDART_INF)) {
      if (threadIdx.x == 0) {
        out.idx[k] = -1;
        out.t[k] = CUDART_INF;
        out.flag[k] = VR_RAY_ESCAPED;
        if (out.rp)
          for (int j = 0; j < D; ++j) out.rp[k * D + j] = CUDART_NAN;
      }
      return;
    }
    double rp[D];
#pragma unroll
    for (int j = 0; j < D; ++j) rp[j] = fma(best, r.u[j], r.x[j]);
    const double radius = sqrt(fmax(fma(best, fma(2.0, r.bu, best), r.base), 0.0));
    double second = CUDART_INF;
    for (int64_t c = threadIdx.x; c < n_cand; c += NT) {
      if ((int)c == bi) continue;
      const double* xc = crec + c * S;
      double q = 0.0, dd = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        q = fma(r.u[j], xc[j], q);
        const double a = rp[j] - xc[j];
        dd = fma(a, a, dd);
      }
      if (q > r.thr) second = fmin(second, sqrt(dd));
    }
    int dummy = 0;
    block_argmin<NT>(second, dummy, sh_t, sh_i);
    if (threadIdx.x == 0) {
      out.idx[k] = cand ? cand[bi] : bi;
      out.t[k] = best;
      if (out.rp)
        for (int j = 0; j < D; ++j) out.rp[k * D + j] = rp[j];
      out.flag[k] = (second < radius * (1.0 + VR_TOL_DEGENERATE)) ? VR_RAY_DEGENERATE : VR_RAY_OK;
    }
  }
}

template <int D, int NT, class Src>
__global__ void __launch_bounds__(NT)
    k_raycast_recheck(Src src, const double* __restrict__ crec, const int32_t* __restrict__ cand,
                      int64_t n_cand, const int32_t* __restrict__ list,
                      const int32_t* __restrict__ count, RayOut out) {
  __shared__ double sh_t[NT / 32];
  __shared__ int sh_i[NT / 32];
  const int cntl = *count;
  for (int li = blockIdx.x; li < cntl; li += gridDim.x)
    recheck_ray<D, NT>(src, list[li], crec, cand, n_cand, out, sh_t, sh_i);
}

// Host-side launch helpers -------------------------------------------------
template <int D, int R_, int MINB_>
struct RaycastCfgT {
  static constexpr int NT = 128;
  static constexpr int R = R_;
  static constexpr int MINB = MINB_;
  static constexpr int TILE = 256;
  static constexpr int STAGES = 4;
  static size_t smem(bool f32) {
    return (size_t)STAGES * TILE *
               (rec_stride(D) * sizeof(double) + (f32 ? rec32_stride(D) * sizeof(float) : 0)) +
           STAGES * (sizeof(uint64_t) + sizeof(int));
  }
};

template <int D>
using RaycastCfg = RaycastCfgT<D, (D <= 3) ? 4 : 2, (D <= 3 || D >= 7) ? 2 : 3>;

// packed-pair fp32 screen (screen_tile_pairs): R rays per thread share each
// loaded candidate pair
#ifndef VR_EX_R
#define VR_EX_R 2
#endif
#ifndef VR_EX_MINB
#define VR_EX_MINB 2
#endif
template <int D>
using RaycastPairsCfg = RaycastCfgT<D, VR_EX_R, VR_EX_MINB>;

// Screening inputs shared by both kernels: fp32 centred records (nullable ->
// fp64 screen) and the frame constants.
struct Screen {
  const float* rec32;   // records matching `crec` (same row order), or nullptr
  const float* rec32p;  // the same rows pair-interleaved (nullable: row layout)
  Frame fr;
};

template <class C, int D, bool F32, class Src, bool PAIRS = false>
int launch_raycast_cfg(const Src& src, int64_t n_rays, const double* crec, const int32_t* cand,
                       int64_t n_cand, const Screen& sc, const RayOut& out, cudaStream_t st) {
  auto kern = k_raycast<D, C::R, C::NT, C::TILE, C::STAGES, C::MINB, F32, Src, PAIRS>;
  const size_t sm = C::smem(F32);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int64_t per_block = (int64_t)C::NT * C::R;
  const int64_t grid = (n_rays + per_block - 1) / per_block;
  kern<<<(unsigned)grid, C::NT, sm, st>>>(src, crec, PAIRS ? sc.rec32p : sc.rec32, cand, n_cand,
                                          sc.fr, out);
  VR_RETURN_LAUNCH();
}

Screen make_screen(double sqmax, const vr_screen32* s32, int d);

// d = 9 .. 16: the exhaustive fp64 screen only (one ray per thread; the
// fp32 / tensor-core / pruned paths are specialised for d <= 8).
template <int D, class Src>
int launch_raycast_fp64(const Src& src, int64_t n_rays, const double* crec, const int32_t* cand,
                        int64_t n_cand, const Screen& sc, const RayOut& out, cudaStream_t st) {
  if (n_rays <= 0) return VR_OK;
  if (n_cand <= 0) return VR_EINVAL;
  if (out.recheck_count) {
    cudaError_t e = cudaMemsetAsync(out.recheck_count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return vr_cuda_status(e);
  }
  return launch_raycast_cfg<RaycastCfgT<D, 1, 1>, D, false>(src, n_rays, crec, cand, n_cand, sc,
                                                             out, st);
}

// Tuning hook: VR_RAYCAST_VARIANT selects alternative register blockings
// for d = 6 (the config-2 shape); 0 = default.
int raycast_variant();

template <int D, class Src>
int launch_raycast(const Src& src, int64_t n_rays, const double* crec, const int32_t* cand,
                   int64_t n_cand, const Screen& sc, const RayOut& out, cudaStream_t st) {
  if (n_rays <= 0) return VR_OK;
  if (n_cand <= 0) return VR_EINVAL;
  if (out.recheck_count) {  // the re-check list is rebuilt by every launch
    cudaError_t e = cudaMemsetAsync(out.recheck_count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return vr_cuda_status(e);
  }
#ifndef VR_NO_EXHAUSTIVE_PAIRS
  if (sc.rec32p)
    return launch_raycast_cfg<RaycastPairsCfg<D>, D, true, Src, true>(src, n_rays, crec, cand,
                                                                      n_cand, sc, out, st);
#endif
  if (sc.rec32)
    return launch_raycast_cfg<RaycastCfg<D>, D, true>(src, n_rays, crec, cand, n_cand, sc, out, st);
  return launch_raycast_cfg<RaycastCfg<D>, D, false>(src, n_rays, crec, cand, n_cand, sc, out, st);
}

struct PrunedIndex {
  const double* crec;      // records in kd-order (padded)
  const float* crec32;     // fp32 centred records in kd-order (nullable)
  const int32_t* perm;     // kd position -> generator index
  const int32_t* inv_perm; // generator index -> kd position
  const double* tile_box;  // ntiles x 2D
  const float* tile_box32; // ntiles x 2D, centred, rounded outward
  const double* node_box;  // kd-tree nodes (heap layout) x 2D
  const float* node_box32;
  const int2* node_range;  // [first tile, last tile + 1) per node
  int64_t n;
  WideTree wide;           // 32-ary tree over the tiles (cooperative kernel)
  const float* crecB;      // tensor-core screen operand (nullable)
  const float* crec32s;    // kd-ordered fp32 centred rows, vr_pack_records32 layout (with crecB)
  const float* node_cb32;  // node boxes as centre / half-extent rows (with crecB)
  const float* crecU;      // tcgen05 screen operand, canonical UMMA layout (nullable)
};

template <int D, class Src>
int launch_pruned_tc(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                     const RayOut& out, cudaStream_t st, unsigned long long* work);

#ifdef VR_PRUNE_TILE_OVERRIDE  // tuning builds only (the Python index must match: VR_PRUNE_TILE)
constexpr int PRUNE_TILE = VR_PRUNE_TILE_OVERRIDE;
#else
constexpr int PRUNE_TILE = 64;
#endif
constexpr int PRUNE_BLOCK = 32;

template <int D, class Src>
int launch_sweep(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                 const RayOut& out, cudaStream_t st, unsigned long long* work);
int sweep_mode();  // VR_SWEEP=1 / 0 forces the tensor-core sweep on / off

template <int D, int R, int MINB, bool F32, class Src, bool MMA = false>
int launch_pruned_rm(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                     const RayOut& out, cudaStream_t st, unsigned long long* work) {
  const int64_t per_block = 32 * R;
  const int64_t items = (n_rays + per_block - 1) / per_block;
  auto kern = k_raycast_pruned<D, R, PRUNE_TILE, PRUNE_BLOCK, MINB, F32, Src, MMA>;
  unsigned long long* next_item = nullptr;
  int64_t grid = items;
#ifdef VR_PERSISTENT
  static int slots = 0;  // resident CTAs on the whole GPU (one warp each)
  if (!slots) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, 0);
    slots = sms * per_sm;
  }
  if (items > slots) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&next_item), sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(next_item, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return vr_cuda_status(e);
    grid = slots;
  }
#endif
  kern<<<(unsigned)grid, 32, 0, st>>>(src, ix.crec, ix.crec32, ix.crecB, ix.crec32s, ix.perm, ix.inv_perm, ix.n,
                                      ix.tile_box, ix.tile_box32, ix.node_box,
                                      MMA ? ix.node_cb32 : ix.node_box32,
                                      ix.node_range, fr, out, work, next_item);
  cudaError_t le = cudaGetLastError();
  if (next_item) cudaFreeAsync(next_item, st);
  return vr_cuda_status(le);
}

int raycast_variant();
int mma_mode();  // VR_MMA=0 disables the tensor-core screen (A/B runs)

template <int D, bool F32, class Src>
int launch_pruned_f(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                    const RayOut& out, cudaStream_t st, unsigned long long* work) {
  if constexpr (D == 6 && F32) {
    switch (raycast_variant()) {
      case 1: return launch_pruned_rm<D, 2, 10, F32>(src, n_rays, ix, fr, out, st, work);
      case 2: return launch_pruned_rm<D, 2, 8, F32>(src, n_rays, ix, fr, out, st, work);
      case 3: return launch_pruned_rm<D, 1, 20, F32>(src, n_rays, ix, fr, out, st, work);
      case 4: return launch_pruned_rm<D, 1, 12, F32>(src, n_rays, ix, fr, out, st, work);
      default: break;
    }
  }
  // one ray per lane: the warp's 32 rays are spatially tighter (fewer tiles
  // pass the union test) and the lighter register file fits 12-24 warps/SM
#ifdef VR_PRUNED_MINB
  constexpr int MINB = VR_PRUNED_MINB;
#else
  constexpr int MINB = (D <= 3) ? 24 : (D <= 4 ? 20 : (D <= 6 ? 16 : 12));
#endif
#ifdef VR_MMA_MINB
  constexpr int MMA_MINB = VR_MMA_MINB;
#else
  constexpr int MMA_MINB = MINB;
#endif
  // tensor-core screen from d = 5 (config 4, d = 4: 0.126 vs 0.118 s with
  // the packed-FFMA2 screen, whose cost scales with d)
#ifndef VR_MMA_MIN_D
#define VR_MMA_MIN_D 5
#endif
  if constexpr (F32 && PRUNE_TILE == 64 && D >= VR_MMA_MIN_D) {
    // 5th-generation tensor cores (tcgen05 + TMEM, 128-ray CTAs): VR_MMA=2
    if (ix.crecU && ix.crec32s && ix.node_cb32 && mma_mode() == 2)
      return launch_pruned_tc<D>(src, n_rays, ix, fr, out, st, work);
    if (ix.crecB && ix.crec32s && ix.node_cb32 && mma_mode() != 0)
      return launch_pruned_rm<D, 1, MMA_MINB, F32, Src, true>(src, n_rays, ix, fr, out, st, work);
  }
  return launch_pruned_rm<D, 1, MINB, F32>(src, n_rays, ix, fr, out, st, work);
}

template <int D, class Src>
int launch_coop(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                const RayOut& out, cudaStream_t st, unsigned long long* work) {
  constexpr int NW = 4;
  constexpr int MINB = VR_COOP_MINB;
  const int64_t grid = (n_rays + NW - 1) / NW;
  if constexpr (PRUNE_TILE == 64) {
    k_raycast_coop<D, PRUNE_TILE, NW, MINB, Src><<<(unsigned)grid, NW * 32, 0, st>>>(
        src, n_rays, ix.crec, ix.crec32, ix.perm, ix.inv_perm, ix.wide, fr, out, work);
    VR_RETURN_LAUNCH();
  }
  return VR_EINVAL;
}

int coop_mode();
int hsweep_mode();  // VR_HSWEEP=1 / 0: the mma.sync sweep on / off (default: auto)

template <int D, class Src>
int launch_hsweep(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                  const RayOut& out, cudaStream_t st, unsigned long long* work) {
  if constexpr (mma_ksteps(D) == 1 && PRUNE_TILE == 64) {
// measured (config 2): 4 warps x 4 stages 3.95 ms; 4 x 6 4.48 ms; 8 x 8
// 4.11 ms; 8 x 12 5.84 ms
#ifndef VR_HSWEEP_NW
#define VR_HSWEEP_NW 4
#endif
#ifndef VR_HSWEEP_MINB
#define VR_HSWEEP_MINB 4
#endif
#ifndef VR_HSWEEP_STAGES
#define VR_HSWEEP_STAGES 4
#endif
    constexpr int NW = VR_HSWEEP_NW, STAGES = VR_HSWEEP_STAGES, TC = 256;
    const int64_t per = (int64_t)NW * 32;
    const int64_t grid = (n_rays + per - 1) / per;
    auto kern = k_raycast_hsweep<D, NW, STAGES, TC, VR_HSWEEP_MINB, Src>;
    const int smem = STAGES * TC * 8 * mma_ksteps(D) * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(src, n_rays, ix.crec, ix.crecB, ix.crec32s, ix.perm,
                                                ix.inv_perm, rec_rows(ix.n), fr, out, work);
    VR_RETURN_LAUNCH();
  }
  return VR_EINVAL;
}

// Host-side view of the C-ABI index -> kernel parameters.
inline PrunedIndex pruned_index_from(const vr_prune_index* ix, bool f32) {
  PrunedIndex pi{ix->rec, f32 ? ix->rec32 : nullptr, ix->perm, ix->inv_perm, ix->tile_box,
                 ix->tile_box32, ix->node_box, ix->node_box32,
                 reinterpret_cast<const int2*>(ix->node_range), ix->n, WideTree{}};
  pi.crecB = f32 ? ix->recB : nullptr;
  pi.crec32s = f32 ? ix->rec32rows : nullptr;
  pi.node_cb32 = f32 ? ix->node_cb32 : nullptr;
  pi.crecU = f32 ? ix->recU : nullptr;
  pi.wide.box32 = ix->wide_box32;
  pi.wide.levels = ix->wide_levels;
  for (int l = 0; l < WIDE_MAX_LEVELS; ++l) {
    pi.wide.off[l] = l < ix->wide_levels ? ix->wide_off[l] : 0;
    pi.wide.cnt[l] = l < ix->wide_levels ? ix->wide_cnt[l] : 0;
  }
  return pi;
}

template <int D, class Src>
int launch_raycast_pruned(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                          const RayOut& out, cudaStream_t st, unsigned long long* work) {
  if (n_rays <= 0) return VR_OK;
  if (ix.n <= 0) return VR_EINVAL;
  if (out.recheck_count) {
    cudaError_t e = cudaMemsetAsync(out.recheck_count, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return vr_cuda_status(e);
  }
  // The cooperative warp-per-ray kernel wins only for sparse, incoherent
  // high-dimensional rays (config-5 sample: 7.2 vs 9.5 ms) and loses on
  // dense traversal levels (config 5 L=5: 10.3 vs 7.4 s) and everywhere at
  // d <= 6.
  // Auto (VR_COOP unset): sparse batches at d >= 7 -- fewer than one ray per
  // 64 generators, e.g. the 10,000 descent rays of config 5 among 1e6
  // generators (0.166 -> 0.126 s for the whole descent) -- and batches too
  // small to fill the GPU with 32-ray warps (< 8192 rays: the small levels
  // of a full traversal; config 1 12.5 -> 10.5 ms) go to the cooperative
  // kernel; VR_COOP=1 / 0 force it on / off.
  if constexpr (PRUNE_TILE == 64 && D <= 6) {
    if (ix.crec32 && ix.crecU && ix.crec32s && sweep_mode() > 0)
      return launch_sweep<D>(src, n_rays, ix, fr, out, st, work);
  }
  if constexpr (mma_ksteps(D) == 1 && PRUNE_TILE == 64) {
    if (ix.crec32 && ix.crecB && ix.crec32s && rec_rows(ix.n) % 256 == 0 && hsweep_mode() > 0)
      return launch_hsweep<D>(src, n_rays, ix, fr, out, st, work);
  }
  const int cm = coop_mode();
  const bool coop = cm > 0 || (cm < 0 && (n_rays < 8192 || (D >= 7 && n_rays * 64 < ix.n)));
  if (ix.crec32 && ix.wide.box32 && ix.wide.levels >= 2 && coop)
    return launch_coop<D>(src, n_rays, ix, fr, out, st, work);
  if (ix.crec32 && ix.tile_box32 && ix.node_box32)
    return launch_pruned_f<D, true>(src, n_rays, ix, fr, out, st, work);
  return launch_pruned_f<D, false>(src, n_rays, ix, fr, out, st, work);
}

template <int D, class Src>
int launch_recheck(const Src& src, int64_t max_list, const double* crec, const int32_t* cand,
                   int64_t n_cand, const int32_t* list, const int32_t* count, const RayOut& out,
                   cudaStream_t st) {
  if (max_list <= 0) return VR_OK;
  const int64_t grid = max_list < 4096 ? max_list : 4096;
  k_raycast_recheck<D, 256, Src><<<(unsigned)grid, 256, 0, st>>>(src, crec, cand, n_cand, list,
                                                                 count, out);
  VR_RETURN_LAUNCH();
}

}  // namespace vr

#include "raycast_tc.cuh"
