// Pruned RayCast with a 5th-generation tensor-core screen (tcgen05 + TMEM).
//
// One CTA = 4 warps = 128 spatially coherent rays (one per thread) sharing ONE
// kd walk.  Per visited tile of 64 candidates the screen of all 128 rays is a
// single tcgen05.mma (M = 128 rays, N = 64 candidates, K = 8 per k-step,
// kind::tf32) issued by one thread:
//     f~ = [z32, 1, ctc] . [x~, |x~|^2, 1]          (sphere product, TMEM cols 0-63)
//     h~ = [u32, 0, c2 ] . [x~, |x~|^2, 1]          (halfspace product, cols 64-127)
// with the same operands and conservative bounds as the mma.sync screen
// (screen_tile_mma, ray_set_best): a pair can matter only if f~ < 0 and
// h~ >= 0.  The accumulators land in TMEM; each thread drains its own ray's
// row (its warp's 32-lane TMEM slice) with tcgen05.ld 32x32b -- no ballots,
// no fragment shuffles -- and OR-reduces the sign bits; the rare pairs go
// through the unchanged fp64 rare path (ray_rare_block), so results are
// bitwise those of every other screen.  Candidate tiles arrive by TMA bulk
// copy in the canonical K-major no-swizzle UMMA layout (vr_pack_records_umma);
// the ray rows are rewritten in shared memory after sphere updates (a stale
// sphere only screens a superset).  The kd walk is decided CTA-wide (a node
// is descended if any of the 128 rays needs it; one barrier per expanded
// node tests both children).
//
// Operand layout (K-major, SWIZZLE_NONE, canonical UMMA "interleave"): an
// 8-row x 16-byte core matrix per (row group g, K chunk q); row m of a k-step
// at byte  s * ROWS * 32 + (m >> 3) * 256 + q * 128 + (m & 7) * 16;
// descriptor LBO (K chunk stride) = 128 B, SBO (row-group stride) = 256 B.
#pragma once

namespace vr {

constexpr int TC_RAYS = 128;  // rays per CTA (tcgen05 M)
constexpr int TC_TILE = 64;   // candidates per tile (tcgen05 N)

__host__ __device__ constexpr int tc_ksteps(int d) { return (d + 2 + 7) / 8; }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  constexpr uint64_t LBO = 128, SBO = 256;
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((LBO >> 4) << 16) | ((SBO >> 4) << 32) |
         (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}

// kind::tf32, D = f32, A = B = tf32, both K-major, N = 64, M = 128
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_TILE >> 3) << 17) |
                              ((uint32_t)(TC_RAYS >> 4) << 24);

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(TC_IDESC), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 consecutive fp32 TMEM columns of this thread's lane -> OR of their bits
// (the sign bit of the result is set iff some value is negative or -0).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Sign bits of 32 values -> a 32-bit mask (bit c = value c < 0, -0 included).
__device__ __forceinline__ uint32_t sign_mask32(const uint32_t (&v)[32]) {
  uint32_t m = 0u;
#pragma unroll
  for (int c = 0; c < 32; ++c) m |= (v[c] >> 31) << c;
  return m;
}

// This thread's operand row (K = 8 KS features) in the canonical layout.
template <int D>
__device__ __forceinline__ void tc_store_row(float* base, int m, const float (&f)[8 * tc_ksteps(D)]) {
#pragma unroll
  for (int s = 0; s < tc_ksteps(D); ++s)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float4* p = reinterpret_cast<float4*>(base + s * TC_RAYS * 8 + (m >> 3) * 64 + q * 32 +
                                            (m & 7) * 4);
      *p = make_float4(f[8 * s + 4 * q], f[8 * s + 4 * q + 1], f[8 * s + 4 * q + 2],
                       f[8 * s + 4 * q + 3]);
    }
}

template <int D>
__device__ __forceinline__ void tc_store_a(const RayState<D>& r, float* sA, int m) {
  float f[8 * tc_ksteps(D)];
#pragma unroll
  for (int k = 0; k < 8 * tc_ksteps(D); ++k)
    f[k] = k < D ? __uint_as_float(tf32_rn(r.z32[k])) : k == D ? 1.0f : k == D + 1 ? r.ctc : 0.0f;
  tc_store_row<D>(sA, m, f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the MMA
}

template <int D>
__device__ __forceinline__ void tc_store_u(const RayState<D>& r, const Frame& fr, float* sU, int m) {
  // as mma_store_u: c2 = bsl32 - thr32 + e_u rounded up (the conservative
  // fp32 halfspace pre-filter, tf32 error bound included)
  const double xm = sqrt(fr.sqmax32);
  const double eu = 1.25 * (9.775161743164062e-04 * xm +
                            1.52587890625e-05 * (xm + fabs((double)r.thr32) + 1.0));
  double c2 = (double)r.bsl32 - (double)r.thr32 + eu;
  c2 = fmin(fmax(c2, -1e30), 1e30);
  float f[8 * tc_ksteps(D)];
#pragma unroll
  for (int k = 0; k < 8 * tc_ksteps(D); ++k)
    f[k] = k < D ? __uint_as_float(tf32_rn(r.u32[k])) : k == D + 1 ? tf32_up(__double2float_ru(c2))
                                                                 : 0.0f;
  tc_store_row<D>(sU, m, f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// CTA-wide DFS over the kd tree (heap layout).  Every thread keeps the same
// stack (decisions are CTA-uniform): slot i in lane i of each warp.
template <int D>
struct CtaCursor {
  int s_node = 0, s_lo = 0, s_hi = 0;
  int sp = 0;
  int64_t st = 0;
  unsigned long long tests = 0;
  __device__ __forceinline__ void push(int node, int2 rg) {
    if (sp >= 32) __trap();
    if ((int)(threadIdx.x & 31) == sp) {
      s_node = node;
      s_lo = rg.x;
      s_hi = rg.y;
    }
    ++sp;
  }
  // bit 0: some ray needs node a, bit 1: node b (one barrier).  Three flag
  // words rotate: test i ORs into word i % 3 and clears word (i + 1) % 3
  // before its barrier; every read of that word (test i - 2) happened before
  // barrier i - 1.
  __device__ __forceinline__ int cta_needs2(const RayState<D>& r, const float* __restrict__ cb32,
                                            int a, int b, int* flags) {
    const bool na = ray_needs_box32_ch<D>(r, cb32 + (int64_t)a * box32_stride(D));
    const bool nb = b >= 0 && ray_needs_box32_ch<D>(r, cb32 + (int64_t)b * box32_stride(D));
    const int slot = (int)(tests % 3);
    ++tests;
    const unsigned ba = __ballot_sync(0xffffffffu, na), bb = __ballot_sync(0xffffffffu, nb);
    if (threadIdx.x == 0) flags[slot == 2 ? 0 : slot + 1] = 0;
    if ((threadIdx.x & 31) == 0 && (ba | bb)) atomicOr(flags + slot, (ba ? 1 : 0) | (bb ? 2 : 0));
    __syncthreads();
    return flags[slot];
  }
  __device__ __forceinline__ void init(int64_t start_tile, const RayState<D>& r,
                                       const float* __restrict__ cb32,
                                       const int2* __restrict__ node_range, int* flags) {
    st = start_tile;
    sp = 0;
    if (cta_needs2(r, cb32, 0, -1, flags) & 1) push(0, __ldg(node_range));
  }
  __device__ __forceinline__ int64_t next(const RayState<D>& r, const float* __restrict__ cb32,
                                          const int2* __restrict__ node_range, int* flags) {
    while (sp > 0) {
      --sp;
      const int node = __shfl_sync(0xffffffffu, s_node, sp);
      const int lo = __shfl_sync(0xffffffffu, s_lo, sp);
      const int hi = __shfl_sync(0xffffffffu, s_hi, sp);
      if (hi - lo == 1) return lo;
      const int l = 2 * node + 1, rr = 2 * node + 2;
      const int2 rl = __ldg(node_range + l), rg = __ldg(node_range + rr);
      const int need = cta_needs2(r, cb32, l, rr, flags);
      if (st < rl.y) {
        if (need & 2) push(rr, rg);
        if (need & 1) push(l, rl);
      } else {
        if (need & 1) push(l, rl);
        if (need & 2) push(rr, rg);
      }
    }
    return -1;
  }
};

template <int D, int MINB, class Src>
__global__ void __launch_bounds__(TC_RAYS, MINB)
    k_raycast_tc(Src src, const double* __restrict__ crec, const float* __restrict__ crecU,
                 const float* __restrict__ crec32s, const int32_t* __restrict__ perm,
                 const int32_t* __restrict__ inv_perm, const float* __restrict__ node_cb32,
                 const int2* __restrict__ node_range, Frame fr, RayOut out,
                 unsigned long long* __restrict__ work) {
  constexpr int S = rec_stride(D);
  constexpr int KS = tc_ksteps(D);
  constexpr uint32_t TILE_BYTES = TC_TILE * 32 * KS;
  __shared__ __align__(1024) float sA[TC_RAYS * 8 * KS];
  __shared__ __align__(1024) float sU[TC_RAYS * 8 * KS];
  __shared__ __align__(1024) float bufB[2][TC_TILE * 8 * KS];
  __shared__ __align__(8) uint64_t bar_tile[2];
  __shared__ __align__(8) uint64_t bar_mma;
  __shared__ uint32_t tmem_base_s;
  __shared__ int flags[3];
  __shared__ int64_t start_tile_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(128u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar_tile[0], 1);
    mbar_init(&bar_tile[1], 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
    flags[0] = flags[1] = flags[2] = 0;
  }
  const int64_t k = (int64_t)blockIdx.x * TC_RAYS + tid;
  RayState<D> ray;
  const bool act = src.load(k, ray, fr);
  if (!act) init_padding_lane<D, 1>(ray);
  if (act) ray.gk = inv_perm[src.gen(k)];
  if (tid == 0) start_tile_s = inv_perm[src.gen((int64_t)blockIdx.x * TC_RAYS)] / TC_TILE;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const int64_t st = start_tile_s;
  const int64_t so = act ? (int64_t)ray.gk / TC_TILE : st;  // the ray's own start tile
  seed_tile32<D>(ray, crec32s + so * TC_TILE * rec32_stride(D), crec + so * TC_TILE * S,
                 (int)(so * TC_TILE), fr);
  tc_store_a<D>(ray, sA, tid);
  tc_store_u<D>(ray, fr, sU, tid);
  CtaCursor<D> cur;
  cur.init(st, ray, node_cb32, node_range, flags);  // (its barrier publishes sA / sU)
  auto issue = [&](int64_t t, int b) {
    if (tid == 0) {
      mbar_arrive_expect_tx(&bar_tile[b], TILE_BYTES);
      bulk_g2s(bufB[b], crecU + t * (TC_TILE * 8 * KS), TILE_BYTES, &bar_tile[b]);
    }
  };
  uint32_t ph_tile = 0u, ph_mma = 0u;
  unsigned long long tiles_done = 0, rare_blocks = 0, entries = 0;
  int b = 0;
  int64_t t = cur.next(ray, node_cb32, node_range, flags);
  if (t >= 0) issue(t, 0);
  const uint32_t row = tmem + ((uint32_t)(warp * 32) << 16);
  while (t >= 0) {
    // walk one step ahead (its barriers also order the previous tile's TMEM
    // reads and A-row updates before this tile's MMA)
    const int64_t tn = cur.next(ray, node_cb32, node_range, flags);
    if (tn >= 0) issue(tn, b ^ 1);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      mbar_wait(&bar_tile[b], (ph_tile >> b) & 1u);
      tc_fence_after();
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const uint64_t bd = umma_desc(smem_u32(bufB[b] + s * TC_TILE * 8));
        umma_tf32(tmem, umma_desc(smem_u32(sA + s * TC_RAYS * 8)), bd, s);
        umma_tf32(tmem + TC_TILE, umma_desc(smem_u32(sU + s * TC_RAYS * 8)), bd, s);
      }
      umma_commit(&bar_mma);
    }
    ph_tile ^= 1u << b;
    mbar_wait(&bar_mma, ph_mma);
    ph_mma ^= 1u;
    tc_fence_after();
    ++tiles_done;
    uint32_t v[32];
    tmem_ld32(row, v);
    tmem_wait_ld();
    uint32_t lo = sign_mask32(v);
    tmem_ld32(row + 32, v);
    tmem_wait_ld();
    uint32_t hi = sign_mask32(v);
    if (__any_sync(0xffffffffu, (lo | hi) != 0u)) {
      // some pair of this warp passed the sphere product: the halfspace
      // product removes the pairs behind the ray (the conservative pre-filter)
      tmem_ld32(row + TC_TILE, v);
      tmem_wait_ld();
      lo &= ~sign_mask32(v);
      tmem_ld32(row + TC_TILE + 32, v);
      tmem_wait_ld();
      hi &= ~sign_mask32(v);
      const int gbase = (int)(t * TC_TILE);
      unsigned long long m = ((unsigned long long)hi << 32) | lo;
      const int rel = ray.ib - gbase;  // the current best itself
      if ((unsigned)rel < 64u) m &= ~(1ull << rel);
      const int relg = ray.gk - gbase;  // g: on every sphere, never valid
      if ((unsigned)relg < 64u) m &= ~(1ull << relg);
      if (m) {
        ++rare_blocks;
        entries += __popcll(m);
        const int nupd0 = ray.nupd;
        const double* tile64 = crec + t * TC_TILE * S;
        if ((unsigned)m) ray_rare_block<D, true>(ray, tile64, (unsigned)m, gbase, fr);
        if ((unsigned)(m >> 32))
          ray_rare_block<D, true>(ray, tile64 + 32 * S, (unsigned)(m >> 32), gbase + 32, fr);
        if (ray.nupd != nupd0) tc_store_a<D>(ray, sA, tid);
      }
    }
    b ^= 1;
    t = tn;
  }
  if (act) ray_store<D>(ray, src.id(k), perm, out);
  if (work) {
    unsigned long long e = entries, rb = rare_blocks, up = act ? ray.nupd : 0;
    for (int off = 16; off > 0; off >>= 1) {
      e += __shfl_xor_sync(0xffffffffu, e, off);
      rb += __shfl_xor_sync(0xffffffffu, rb, off);
      up += __shfl_xor_sync(0xffffffffu, up, off);
    }
    if ((tid & 31) == 0) {
      atomicAdd(work + 1, rb);
      atomicAdd(work + 3, e);
      atomicAdd(work + 4, up);
    }
    if (tid == 0) {
      atomicAdd(work, tiles_done * (unsigned long long)(TC_TILE * TC_RAYS));
      atomicAdd(work + 5, cur.tests);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128u));
  }
}

template <int D, class Src>
int launch_pruned_tc(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                     const RayOut& out, cudaStream_t st, unsigned long long* work) {
  const int64_t grid = (n_rays + TC_RAYS - 1) / TC_RAYS;
  k_raycast_tc<D, 4, Src><<<(unsigned)grid, TC_RAYS, 0, st>>>(
      src, ix.crec, ix.crecU, ix.crec32s, ix.perm, ix.inv_perm, ix.node_cb32, ix.node_range, fr,
      out, work);
  VR_RETURN_LAUNCH();
}


// ---------------------------------------------------------------------------
// Sweep kernel: the tensor-core screen of EVERY generator for 128 rays per
// CTA, no kd walk (small N at d <= 6, e.g. config 2: N = 20,000).  The warp
// kernels spend their time in the tree walk and its divergent decisions;
// here one thread issues a single tcgen05.mma of M = 128 rays x N = NB
// candidates (K = 8: [z32, 1, ctc] . [x~, |x~|^2, 1], the same operands and
// conservative bound as k_raycast_tc) per step, into one of two TMEM
// accumulators, while the four warps drain the other one: each thread
// tcgen05.ld's its ray's NB results and ORs their sign bits (~0.5 LOP3 per
// pair).  The rare pairs go through the unchanged fp64 rare path
// (ray_rare_block), so results are bitwise those of every other screen.
//
// Pipeline (thread 0 issues TMA and MMA; all 128 threads drain):
//   step j:  issue MMA j+1 (A[(j+1)&1], B stage (j+1)%ST) -> TMEM[(j+1)&1]
//            wait MMA j; refill B stage j%ST with block j+ST
//            drain TMEM[j&1]; rare path; rewrite A[j&1] rows of rays whose
//            sphere moved in this or the previous step
//            barrier (TMEM[j&1] drained and A[j&1] written before MMA j+2)
// A ray's row is rewritten into both buffers over two steps after an update,
// so an MMA reads either the current or an older (larger) sphere: stale
// spheres screen a superset, which keeps the screen conservative.
// Blocks of NB candidates are visited in a spiral around the CTA's home
// block (the kd tile of its first ray's generator): the rays' spheres shrink
// within the first few steps and the remaining blocks rarely hit.
// ---------------------------------------------------------------------------
constexpr int SWEEP_RAYS = 128;
constexpr int SWEEP_STAGES = 4;

__host__ __device__ constexpr uint32_t sweep_idesc(int nb) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(nb >> 3) << 17) |
         ((uint32_t)(SWEEP_RAYS >> 4) << 24);
}

template <int NB>
__device__ __forceinline__ void umma_tf32_n(uint32_t d_tmem, uint64_t a, uint64_t b) {
  asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 0;" ::"r"(d_tmem), "l"(a),
               "l"(b), "r"(sweep_idesc(NB))
               : "memory");
}

__device__ __forceinline__ uint32_t or32(const uint32_t (&v)[32]) {
  uint32_t a = v[0] | v[1] | v[2], b = v[3] | v[4] | v[5], c = v[6] | v[7] | v[8];
  uint32_t e = v[9] | v[10] | v[11], f = v[12] | v[13] | v[14], g = v[15] | v[16] | v[17];
  uint32_t h = v[18] | v[19] | v[20], i = v[21] | v[22] | v[23], j = v[24] | v[25] | v[26];
  uint32_t k = v[27] | v[28] | v[29], l = v[30] | v[31];
  return (a | b | c) | (e | f | g) | (h | i | j) | (k | l);
}

// The sweep screens with ONE product per ray: the sphere row [z32, 1, ctc]
// once the ray has a best candidate, before that the negated halfspace row
// [-u32, 0, -c2] (f~ = -(u~.x~ + c2) < 0 iff the candidate may lie in front,
// the conservative pre-filter of tc_store_u), so a ray whose seed found
// nothing sends only the candidates ahead of it to the rare path.
template <int D>
__device__ __forceinline__ void sweep_store_a(const RayState<D>& r, const Frame& fr, float* sA,
                                              int m, bool act) {
  if (r.ib >= 0 || !act) {
    tc_store_a<D>(r, sA, m);
    return;
  }
  const double xm = sqrt(fr.sqmax32);
  const double eu = 1.25 * (9.775161743164062e-04 * xm +
                            1.52587890625e-05 * (xm + fabs((double)r.thr32) + 1.0));
  double c2 = (double)r.bsl32 - (double)r.thr32 + eu;
  c2 = fmin(fmax(c2, -1e30), 1e30);
  float f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k)
    f[k] = k < D ? -__uint_as_float(tf32_rn(r.u32[k]))
                 : k == D + 1 ? -tf32_up(__double2float_ru(c2)) : 0.0f;
  tc_store_row<D>(sA, m, f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int D, int NB, int MINB, class Src>
__global__ void __launch_bounds__(SWEEP_RAYS, MINB)
    k_raycast_sweep(Src src, const double* __restrict__ crec, const float* __restrict__ crecU,
                    const float* __restrict__ crec32s, const int32_t* __restrict__ perm,
                    const int32_t* __restrict__ inv_perm, int64_t n_rows, Frame fr, RayOut out,
                    unsigned long long* __restrict__ work) {
  static_assert(tc_ksteps(D) == 1, "sweep kernel: one k-step (d <= 6)");
  static_assert(NB % 64 == 0 && NB <= 256, "NB: whole 64-row tiles");
  constexpr int S = rec_stride(D);
  constexpr uint32_t BLK_BYTES = NB * 32;
  __shared__ __align__(1024) float sA[2][SWEEP_RAYS * 8];
  __shared__ __align__(1024) float sB[SWEEP_STAGES][NB * 8];
  __shared__ __align__(8) uint64_t bar_b[SWEEP_STAGES];
  __shared__ __align__(8) uint64_t bar_mma[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ int64_t home_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"((uint32_t)(2 * NB)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const int64_t nblk = n_rows / NB;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < SWEEP_STAGES; ++i) mbar_init(&bar_b[i], 1);
    mbar_init(&bar_mma[0], 1);
    mbar_init(&bar_mma[1], 1);
    fence_mbar_init();
    home_s = (int64_t)inv_perm[src.gen((int64_t)blockIdx.x * SWEEP_RAYS)] / NB;
  }
  const int64_t k = (int64_t)blockIdx.x * SWEEP_RAYS + tid;
  RayState<D> ray;
  const bool act = src.load(k, ray, fr);
  if (!act) init_padding_lane<D, 1>(ray);
  if (act) ray.gk = inv_perm[src.gen(k)];
  if (act) {
    const int64_t so = (int64_t)ray.gk / TC_TILE;  // the ray's own tile
    seed_tile32<D>(ray, crec32s + so * TC_TILE * rec32_stride(D), crec + so * TC_TILE * S,
                   (int)(so * TC_TILE), fr);
  }
  sweep_store_a<D>(ray, fr, sA[0], tid, act);
  sweep_store_a<D>(ray, fr, sA[1], tid, act);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  const int64_t home = home_s;
  auto block_of = [&](int64_t j) -> int64_t {  // spiral: home, +1, -1, +2, -2, ...
    const int64_t off = (j & 1) ? (j + 1) >> 1 : -(j >> 1);
    int64_t b = (home + off) % nblk;
    return b < 0 ? b + nblk : b;
  };
  auto issue_b = [&](int64_t j) {
    const int st = (int)(j % SWEEP_STAGES);
    mbar_arrive_expect_tx(&bar_b[st], BLK_BYTES);
    bulk_g2s(sB[st], crecU + block_of(j) * (NB * 8), BLK_BYTES, &bar_b[st]);
  };
  auto issue_mma = [&](int64_t j) {
    const int st = (int)(j % SWEEP_STAGES);
    mbar_wait(&bar_b[st], (uint32_t)((j / SWEEP_STAGES) & 1));
    tc_fence_after();
    umma_tf32_n<NB>(tmem + (uint32_t)((j & 1) * NB), umma_desc(smem_u32(sA[j & 1])),
                    umma_desc(smem_u32(sB[st])));
    umma_commit(&bar_mma[j & 1]);
  };
  if (tid == 0) {
    for (int64_t j = 0; j < SWEEP_STAGES && j < nblk; ++j) issue_b(j);
    issue_mma(0);
  }
  const uint32_t row = tmem + ((uint32_t)(warp * 32) << 16);
  unsigned long long rare_blocks = 0, entries = 0, rare_steps = 0;
  int dirty = 0;
  for (int64_t j = 0; j < nblk; ++j) {
    if (tid == 0 && j + 1 < nblk) issue_mma(j + 1);
    mbar_wait(&bar_mma[j & 1], (uint32_t)((j >> 1) & 1));
    tc_fence_after();
    if (tid == 0 && j + SWEEP_STAGES < nblk) issue_b(j + SWEEP_STAGES);  // stage j free
    const uint32_t acc = row + (uint32_t)((j & 1) * NB);
    uint32_t any = 0u;
#pragma unroll
    for (int q = 0; q < NB / 32; ++q) {
      uint32_t v[32];
      tmem_ld32(acc + 32 * q, v);
      tmem_wait_ld();
      any |= or32(v);
    }
    const int64_t b = block_of(j);
    const int gb = (int)(b * NB);
    if (__any_sync(0xffffffffu, (int)(any >> 31))) {
      ++rare_steps;
      const int nupd0 = ray.nupd;
#pragma unroll 1
      for (int q = 0; q < NB / 32; ++q) {
        uint32_t v[32];
        tmem_ld32(acc + 32 * q, v);
        tmem_wait_ld();
        uint32_t m = sign_mask32(v);
        const int base = gb + 32 * q;
        const int rel = ray.ib - base;  // the current best itself
        if ((unsigned)rel < 32u) m &= ~(1u << rel);
        const int relg = ray.gk - base;  // g: on every sphere, never valid
        if ((unsigned)relg < 32u) m &= ~(1u << relg);
        if (m) {
          ++rare_blocks;
          entries += __popc(m);
          ray_rare_block<D, true>(ray, crec + (int64_t)base * S, m, base, fr);
        }
      }
      if (ray.nupd != nupd0) dirty = 2;
    }
    if (dirty) {
      sweep_store_a<D>(ray, fr, sA[j & 1], tid, act);
      --dirty;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (act) ray_store<D>(ray, src.id(k), perm, out);
  if (work) {
    unsigned long long e = entries, rb = rare_blocks, up = act ? ray.nupd : 0, a = act ? 1 : 0;
    for (int off = 16; off > 0; off >>= 1) {
      e += __shfl_xor_sync(0xffffffffu, e, off);
      rb += __shfl_xor_sync(0xffffffffu, rb, off);
      up += __shfl_xor_sync(0xffffffffu, up, off);
      a += __shfl_xor_sync(0xffffffffu, a, off);
    }
    if ((tid & 31) == 0) {
      atomicAdd(work, a * (unsigned long long)n_rows);
      atomicAdd(work + 1, rb);
      atomicAdd(work + 2, rare_steps);  // warp steps that entered the rare path
      atomicAdd(work + 3, e);
      atomicAdd(work + 4, up);
    }
#ifdef VR_RARE_STATS
    int stv[5] = {ray.st_out, ray.st_self, ray.st_behind, ray.st_band, ray.st_imp};
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      unsigned long long v = act ? stv[q] : 0;
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if ((tid & 31) == 0) atomicAdd(work + 6 + q, v);
    }
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"((uint32_t)(2 * NB)));
  }
}

template <int D, class Src>
int launch_sweep(const Src& src, int64_t n_rays, const PrunedIndex& ix, const Frame& fr,
                 const RayOut& out, cudaStream_t st, unsigned long long* work) {
  if constexpr (tc_ksteps(D) == 1) {
#ifndef VR_SWEEP_NB
#define VR_SWEEP_NB 128
#endif
    constexpr int NB = VR_SWEEP_NB;
    const int64_t grid = (n_rays + SWEEP_RAYS - 1) / SWEEP_RAYS;
    k_raycast_sweep<D, NB, (NB <= 128 ? 2 : 1), Src><<<(unsigned)grid, SWEEP_RAYS, 0, st>>>(
        src, ix.crec, ix.crecU, ix.crec32s, ix.perm, ix.inv_perm, rec_rows(ix.n), fr, out, work);
    VR_RETURN_LAUNCH();
  }
  return VR_EINVAL;
}

}  // namespace vr
