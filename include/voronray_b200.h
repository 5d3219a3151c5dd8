/*
 * voronray_b200.h -- C ABI of the B200-native incircle RayCast library.
 *
 * The reference (`voronray`, pure Python + numpy/scipy) has no FFI layer: its
 * drop-in boundary is the public Python API (pkg/src/voronray/__init__.py:3-32).
 * Every entry point below replaces one inner operation of that API; the
 * reference function each one stands in for is cited per declaration.
 *
 * Conventions (all entry points):
 *   - plain device pointers + sizes, no framework types;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - stream-ordered, reentrant across streams, no persistent allocation
 *     (callers pass workspaces), no host synchronisation unless stated;
 *   - return 0 (VR_OK) or a negative vr_status / -(1000 + cudaError_t).
 *   - generator indices are 0-based int32 (reference core.py:7).
 *
 * Per-ray flags (uint8):  0 VR_RAY_OK, 1 VR_RAY_ESCAPED (reference: `None`,
 *   raycast.py:190-191), 2 VR_RAY_RECHECK (internal; resolved by
 *   vr_raycast_recheck), 3 VR_RAY_DEGENERATE (reference raises
 *   DegenerateConfiguration, raycast.py:216-219).
 */
#ifndef VORONRAY_B200_H
#define VORONRAY_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum vr_status {
  VR_OK = 0,
  VR_EINVAL = -1,         /* bad size / null pointer / unsupported d          */
  VR_EDIM = -2,           /* d outside [2, 8]                                 */
  VR_ECAPACITY = -3,      /* a caller-sized workspace / table is too small    */
  VR_ECUDA_BASE = -1000   /* -(1000 + cudaError_t)                            */
};

enum vr_ray_flag {
  VR_RAY_OK = 0,
  VR_RAY_ESCAPED = 1,
  VR_RAY_RECHECK = 2,
  VR_RAY_DEGENERATE = 3
};

/* MC per-cell status (reference integrate_mc.py:63-64,184-187). */
enum vr_cell_status {
  VR_CELL_OK = 0,
  VR_CELL_UNBOUNDED = 1,   /* reference raises UnboundedRay(cell, direction)   */
  VR_CELL_DEGENERATE = 2,  /* reference raises DegenerateConfiguration         */
  VR_CELL_OVERFLOW = 3     /* more distinct hit faces than area slots          */
};

int vr_abi_version(void); /* 7 */
const char* vr_status_string(int status);

/* Record stride (doubles) of one packed generator for dimension d:
 * [x_0 .. x_{d-1}, |x|^2, pad] rounded up to an even count (16-B rows). */
int vr_record_stride(int d);

/* Rows of a packed record array for n generators: n rounded up to a
 * multiple of 512.  Rows >= n are sentinels [0, .., 0, +inf] that can never
 * win a RayCast, so every shared-memory tile the kernels stage is full. */
int64_t vr_record_rows(int64_t n);

/* Pack an (n, d) fp64 row-major point array into 16-B aligned records
 * [x, |x|^2, pad] plus the sentinel rows.  Replaces the NodeSet fp64 copy +
 * squared norms (reference core.py:44-51).  rec must hold
 * vr_record_rows(n) * vr_record_stride(d) doubles.  Every `rec` / `cand_rec`
 * argument below uses this padded layout. */
int vr_pack_generators(const double* pts, int64_t n, int d, double* rec,
                       double* sqmax_out /* device, 1 double */, void* stream);

/* Optional fp32 screening input.  The kernels screen every (ray, generator)
 * pair in fp32 in a frame centred at `center` with a rigorous, rounded-up
 * error bound, and send every candidate the fp32 screen cannot exclude
 * through the unchanged fp64 path (fp64 test first) -- results are identical
 * to the fp64 screen.  `rec` holds vr_record_rows(n) rows of
 * vr_record32_stride(d) floats [x - center, |x - center|^2, pad] in the SAME
 * row order as the fp64 records the call scans (sentinel rows: |.|^2 = +inf);
 * sqmax = max |x - center|^2.  NULL selects the fp64 screen. */
typedef struct vr_screen32 {
  const float* rec;
  double center[8];
  double sqmax;
  double bound;   /* max_k |x_k - center_k| over the generators */
  const float* rec_pairs; /* optional: the same rows pair-interleaved
                             (vr_pack_records32_pairs); enables the packed
                             FFMA2 screen of vr_raycast_batch / vr_mc_rays */
} vr_screen32;

int vr_record32_stride(int d);

/* fp32 centred copy of packed fp64 records (same rows, sentinels kept). */
int vr_pack_records32(const double* rec, int64_t rows, int d, const double* center,
                      float* rec32, void* stream);

/* Pair-interleaved copy of vr_pack_records32's rows for the pruned kernel
 * (vr_prune_index.rec32): rows/2 pairs of (2d+5)&~3 floats
 * [x_0a x_0b .. x_{d-1}a x_{d-1}b |.|^2_a |.|^2_b pad]; rows must be even
 * (vr_record_rows is a multiple of 512). */
int vr_pack_records32_pairs(const float* rec32, int64_t rows, int d, float* out,
                            void* stream);

/* fp32 centred records (vr_pack_records32 layout) -> the tensor-core screen
 * operand of the pruned kernel (vr_prune_index.recB): features
 * [x_0 .. x_{d-1}, |x|^2, 1, 0 ..] (sentinel |x|^2 -> 1e30) in KS = ceil((d+2)/8)
 * k-steps of 8; per tile of 64 rows, 8 blocks of 8 candidates, per block KS
 * steps of 32 lanes x 2 tf32 values, lane l holding features 8s + (l & 3) and
 * 8s + (l & 3) + 4 of candidate 8 * block + (l >> 2).  `out` holds
 * rows * 8 * KS floats; rows must be a multiple of 64. */
int vr_pack_records_mma(const float* rec32, int64_t rows, int d, float* out, void* stream);

/* fp32 centred records -> the tcgen05 screen operand (vr_prune_index.recU):
 * the features of vr_pack_records_mma in the canonical UMMA layout;
 * `out` holds rows * 8 * ceil((d+2)/8) floats; rows a multiple of 64. */
int vr_pack_records_umma(const float* rec32, int64_t rows, int d, float* out, void* stream);

/* Batched incircle RayCast (reference raycast_incircle, raycast.py:154-224,
 * with its filtered NN probe _Probe, raycast.py:85-151, core.py:62-103).
 *
 * Ray k starts at x[k*d..] (equidistant to its eta generators), travels along
 * unit u[k*d..], and carries eta[k*eta_len .. +eta_len] (eta_len in [1, d]).
 * Candidate i is valid iff u.x_i > max_{e in eta} u.x_e + 1e-12*max(1,|.|)
 * (raycast.py:95-96, 110-117); the result is the valid i minimising
 * t_i = (|x_i-x|^2 - |x_g-x|^2) / (2 u.(x_i-x_g)), g = eta[0] (raycast.py:203),
 * smallest index on ties, or ESCAPED when no candidate is valid.
 *
 * cand (nullable, n_cand entries, ascending or not) restricts the search to a
 * subset like the reference `candidates=` argument (raycast.py:100-102);
 * cand_rec must then hold the packed records of exactly those generators.
 *
 * Outputs: out_idx (global generator index, -1 on escape), out_t (ray
 * parameter from the reference's centred formula), out_rp (nullable; x+t*u),
 * out_flag.  Rays left in VR_RAY_RECHECK must be passed through
 * vr_raycast_recheck (done internally by vr_raycast_resolve).
 * recheck_list/recheck_count: workspace (n_rays int32 + 1 int32, device),
 * receives the ids of RECHECK rays (the count is zeroed on `stream` first);
 * may be NULL if the caller does not resolve. */
int vr_raycast_batch(const double* rec, int64_t n_gen, int d, double sqmax,
                     const vr_screen32* s32,
                     const double* cand_rec, const int32_t* cand, int64_t n_cand,
                     const double* x, const double* u,
                     const int32_t* eta, int eta_len, int64_t n_rays,
                     int32_t* out_idx, double* out_t, double* out_rp,
                     uint8_t* out_flag, int32_t* recheck_list,
                     int32_t* recheck_count, void* stream);

/* ---- Exact candidate pruning ---------------------
 * Generators reordered by a balanced kd partition into tiles of
 * VR_PRUNE_TILE records (padded with sentinels).  The kd tree over tiles is
 * stored in heap layout (node i -> children 2i+1, 2i+2; a node covering n > 1
 * tiles [lo, hi) splits at lo + n/2), each node with an axis-aligned box.  A
 * warp of spatially coherent rays descends a node only if some ray needs it:
 * a subtree is skipped when, for every ray of the warp, its box lies behind
 * the ray's forward halfspace or outside its current candidate sphere plus
 * the degeneracy/rounding band -- a certificate that no skipped generator
 * could change the result, so the output equals vr_raycast_batch's. */
#define VR_PRUNE_TILE 64
typedef struct vr_prune_index {
  const double* rec;       /* kd-ordered records, vr_record_rows(n) rows       */
  const float* rec32;      /* kd-ordered fp32 centred records, pair-interleaved
                              (vr_pack_records32_pairs); nullable             */
  const int32_t* perm;     /* kd position -> generator index (n)               */
  const int32_t* inv_perm; /* generator index -> kd position (n)               */
  const double* tile_box;  /* ceil(n/64) x 2d, [lo_0..lo_{d-1}, hi_0..]        */
  const float* tile_box32; /* same boxes, centred at vr_screen32.center, fp32
                              rounded outward (lo down, hi up), rows padded
                              to (2d+3)&~3 floats; nullable                  */
  const double* node_box;  /* kd-tree node boxes, heap layout, x 2d            */
  const float* node_box32; /* centred fp32 outward copies; nullable            */
  const int32_t* node_range; /* 2 per node: first tile, last tile + 1        */
  int64_t n;
  /* 32-ary tree over the tiles (cooperative warp-per-ray kernel): level 0 is
   * the tiles themselves (boxes = tile_box32 rows), node j of level l covers
   * nodes [32j, 32j+32) of level l-1; the top level holds one node.  Rows of
   * box32 layout, level l at rows [wide_off[l], wide_off[l] + wide_cnt[l]).
   * wide_box32 == NULL or wide_levels < 2 disables the cooperative kernel. */
  const float* wide_box32;
  int32_t wide_levels;
  int64_t wide_off[8];
  int64_t wide_cnt[8];
  /* Tensor-core screen operand (vr_pack_records_mma): the rec32 rows
   * in mma.sync m16n8k8 B-fragment order, tf32-rounded.  Nullable: without it
   * the pruned kernel screens with packed FFMA2 on rec32. */
  const float* recB;
  /* The kd-ordered fp32 centred rows in vr_pack_records32 layout (the
   * tensor-core kernel's seed pass); required with recB. */
  const float* rec32rows;
  /* The node boxes of node_box32 as centre / half-extent rows [c, h] (same
   * stride; [c - h, c + h] contains the exact box), read by the tensor-core
   * kernel's tree walk; required with recB. */
  const float* node_cb32;
  /* tcgen05 screen operand (vr_pack_records_umma; nullable): the fp32 rows
   * as tf32 features [x, |x|^2, 1, 0 ..] per tile of 64 in the canonical
   * K-major no-swizzle UMMA layout -- per k-step of 8 features, 8-row x
   * 16-byte core matrices: float index s*512 + (c >> 3)*64 + q*32 + (c & 7)*4
   * + e for candidate c, feature 8s + 4q + e. */
  const float* recU;
} vr_prune_index;

/* vr_raycast_batch through the pruned index.  `order` (nullable, n_rays
 * int32) is the processing order: slot k handles ray order[k]; callers sort
 * rays by the kd position of eta[0] so that a warp's rays are spatially
 * coherent.  Outputs are written at the ray's own index.  With s32 != NULL and
 * ix->rec32 != NULL the screen runs in fp32 (s32->rec is not used here).  `work`
 * (nullable, >= VR_WORK_COUNTERS device uint64, zeroed by the caller)
 * accumulates work counters: [0] (ray, generator) pairs screened (32 lanes x
 * 64 per tile), [1] screening blocks with rare work, [2] warp-level rare
 * iterations, [3] rare entries, [4] sphere updates, [5] tree-node tests;
 * builds with VR_RARE_STATS also use [6..10]. */
#define VR_WORK_COUNTERS 16
int vr_raycast_pruned(const double* rec, int64_t n_gen, int d, double sqmax,
                      const vr_screen32* s32, const vr_prune_index* ix, const double* x, const double* u,
                      const int32_t* eta, int eta_len, int64_t n_rays,
                      const int32_t* order, int32_t* out_idx, double* out_t,
                      double* out_rp, uint8_t* out_flag, int32_t* recheck_list,
                      int32_t* recheck_count, uint64_t* work, void* stream);

/* Processing-order keys for the pruned kernels: keys[k] = base * 256 + the
 * direction class of u[k] (signed index of the largest and second-largest
 * |u_j|), base = inv_perm[eta[k * eta_len]] (kd position of the reference
 * generator) or, with eta == NULL, k / rays_per_cell (MC).  Sorting the keys
 * (stable) gives the `order` argument of vr_raycast_pruned / vr_mc_rays_pruned. */
int vr_ray_keys(const int32_t* inv_perm, const int32_t* eta, int eta_len,
                int64_t rays_per_cell, const double* u, int64_t n, int d, int64_t* keys,
                void* stream);

/* The processing order itself: the keys of vr_ray_keys (32-bit when
 * n_base * 256 < 2^32; n_base = the range of base, i.e. n_gen or the cell
 * count) sorted by a stable LSD radix sort, order[k] = ray id of slot k.
 * Call with workspace == NULL to receive the workspace size in
 * *workspace_bytes; otherwise *workspace_bytes is the size passed. */
int vr_ray_order(const int32_t* inv_perm, const int32_t* eta, int eta_len,
                 int64_t rays_per_cell, const double* u, int64_t n, int d, int64_t n_base,
                 int32_t* order, void* workspace, int64_t* workspace_bytes, void* stream);

/* ---- Native build of the pruned index ------------------------------------
 * Replaces the spatial index the reference builds inside NodeSet.__init__
 * (core.py:52-57: scipy cKDTree, used by the kd-tree NN probe core.py:92-103).
 *
 * vr_screen32_stats: the fp32 screening frame of n packed records (the
 *   vr_screen32 fields): stats[0..7] = centre (the bounding-box midpoint, or
 *   `center` (device, d doubles) when given), stats[8] = max |x - c|^2,
 *   stats[9] = max_k |x_k - c_k|.  `stats` is 32 device doubles (16..31 are
 *   scratch).  Read it back once to fill a vr_screen32.
 * vr_prune_index_layout: device bytes of the index arena and of the build
 *   workspace for n generators (flags: VR_PRUNE_MMA also packs recB, the
 *   tensor-core screen operand used from d = 5), tile / node / 32-ary level
 *   counts.
 * vr_build_prune_index: balanced kd partition (per depth: node bounding
 *   boxes, widest axis, stable radix sort of the coordinate + a stable sort
 *   by segment; a node of > 1 tiles splits after floor(tiles / 2) whole
 *   tiles), the kd-ordered records with sentinel rows, perm / inv_perm, tile
 *   / node / 32-ary boxes (fp64 + outward fp32 rows in the frame centred at
 *   `center`, device d doubles: vr_screen32_stats of the generators) and the
 *   fp32 / pair / tensor-core screening copies, all inside `arena`; fills
 *   *out (host struct) with pointers into it.  Stream-ordered, no sync. */
typedef struct vr_prune_layout {
  int64_t arena_bytes;
  int64_t workspace_bytes;
  int64_t n_tiles;
  int64_t n_nodes;
  int32_t wide_levels;
} vr_prune_layout;
#define VR_PRUNE_MMA 1   /* also pack recB (mma.sync screen operand)  */
#define VR_PRUNE_UMMA 2  /* also pack recU (tcgen05 screen operand)   */
int vr_screen32_stats(const double* rec, int64_t n, int d, const double* center, double* stats,
                      void* stream);
int vr_prune_index_layout(int64_t n, int d, int flags, vr_prune_layout* out);
int vr_build_prune_index(const double* rec, int64_t n, int d, const double* center, int flags,
                         void* arena, int64_t arena_bytes, void* workspace,
                         int64_t workspace_bytes, vr_prune_index* out, void* stream);

/* Exact re-evaluation of the rays listed in recheck_list[0 .. *count)
 * (count read on device): centred t for every candidate, argmin with the
 * smallest-index tie-break, then the reference's runner-up degeneracy band
 * second < radius*(1+1e-10) (raycast.py:211-219).  max_list bounds the
 * launch (pass n_rays). */
int vr_raycast_recheck(const double* rec, int64_t n_gen, int d,
                       const double* cand_rec, const int32_t* cand, int64_t n_cand,
                       const double* x, const double* u,
                       const int32_t* eta, int eta_len,
                       const int32_t* recheck_list, const int32_t* recheck_count,
                       int64_t max_list,
                       int32_t* out_idx, double* out_t, double* out_rp,
                       uint8_t* out_flag, void* stream);

/* Filtered nearest neighbour for a batch of queries (reference
 * NodeSet.nearest / nearest2, core.py:62-142): smallest squared distance
 * (expanded form, smallest index on ties, core.py:81-90), skip mask per
 * generator (nullable, uint8, 1 = excluded).  out_d1/out_d2 are the clean
 * Euclidean distances of the nearest and second-nearest (inf if absent),
 * out_idx -1 when every generator is skipped. */
int vr_nearest_batch(const double* rec, int64_t n_gen, int d,
                     const double* q, int64_t n_q, const uint8_t* skip,
                     int32_t* out_idx, double* out_d1, double* out_d2,
                     void* stream);

/* Vertex invariants (reference verify_vertex, core.py:279-296) for a batch:
 * equidistance within tol*rad and no foreign generator closer than
 * rad*(1-tol).  sigma is (n_v, d+1) int32, r is (n_v, d) fp64.
 * out_ok[v] = 1 when both hold. */
int vr_verify_vertices(const double* rec, int64_t n_gen, int d,
                       const int32_t* sigma, const double* r, int64_t n_v,
                       double tol, uint8_t* out_ok, void* stream);

/* fp64 circumcentres of generator tuples (reference graph.py:163-171 and
 * SURVEY.md §8(c) rule 3): solve 2(x_s - x_s0).y = |x_s - x_s0|^2 with
 * partial-pivot LU in registers, r = x_s0 + y.  out_ok = 0 when singular. */
int vr_circumcenters(const double* rec, int d, const int32_t* sigma,
                     int64_t n_v, double* out_r, uint8_t* out_ok, void* stream);

/* Descent directions (graph.py:46-85): for each of n starts with sigma
 * (n, d+1) holding k[i] valid entries, the two-pass modified Gram-Schmidt
 * basis of x_sigma[j] - x_sigma[0] (j = 1 .. k-1; raycast.py:295-308) and
 * the component out_v of the drawn normal z (n, d) orthogonal to it (two
 * passes, raycast.py:311-317), its norm out_nrm, and out_bad = 1 where the
 * rows are affinely dependent (|v| < tol * max(|v0|, 1)). */
int vr_descent_directions(const double* rec, int d, const int32_t* sigma, const int32_t* k,
                          const double* z, int64_t n, double tol, double* out_v,
                          double* out_nrm, uint8_t* out_bad, void* stream);

/* Outward edge directions of vertices (reference _vertex_directions,
 * raycast.py:345-378): column k-1 of -D^{-1} (k>0) or the row sums of D^{-1}
 * (k=0), D rows x_s - x_s0, normalised.  out_u is (n_v, d+1, d);
 * out_ok[v*(d+1)+k] = 0 on a singular / non-finite direction. */
int vr_vertex_directions(const double* rec, int d, const int32_t* sigma,
                         int64_t n_v, double* out_u, uint8_t* out_ok,
                         void* stream);

/* ---- Monte-Carlo cell volumes / interface areas (reference mc_areas_only,
 *      integrate_mc.py:124-161, _mc_areas_batch :164-197) -------------------
 *
 * Rays: n_cells cells (cells[c] = generator index) x rays_per_cell rays.
 * Directions come either from `dirs` ((n_cells*rays_per_cell, d) fp64, raw
 * Gaussian draws normalised on device exactly as sample_unit_sphere,
 * integrate_mc.py:51-56) or, when dirs == NULL, from the Philox4x32-10
 * stream keyed by `seed` with counter (ray, cell, block) + Box-Muller.
 *
 * vr_mc_rays writes per-ray hit index / t / flag (same meaning as the
 * RayCast outputs).  vr_mc_reduce then forms, per cell, in ray order:
 *   length = |(x_c + t y) - x_c|, w = length^(d-1)/cos(n_cj, y),
 *   area[j] = sum w * S_{d-1}/n, volume = sum length^d * S_{d-1}/(d n)
 * (integrate_mc.py:150-160), with areas as a per-cell list of (j, area)
 * sorted by j in slots [c*max_faces, c*max_faces + out_nfaces[c]).
 * out_status[c] / out_first_bad[c] report the first escaping (UnboundedRay)
 * or degenerate ray of the cell in ray order; degenerate rays count only when
 * degenerate_is_error (the per-ray path raises, the neighbour-batch path
 * _mc_areas_batch takes the plain argmin).  surf = S_{d-1} as computed by the
 * caller (integrate_mc.py:44-48).  Face counts are unbounded like the
 * reference's dict (integrate_mc.py:147-160): the per-cell face map holds
 * 2 max_faces slots (at least 1024) in shared memory, or, past 160 KB, in
 * `map_ws` (device, vr_mc_map_bytes bytes; NULL otherwise); a cell with more
 * than max_faces faces reports VR_CELL_OVERFLOW and is re-reduced by the
 * caller with a larger max_faces (faces <= rays and <= n_gen - 1).
 * cell_sel (nullable, n_sel int32 row indices): reduce only those cell rows,
 * block b writing output row b (the overflow re-run). */
int vr_mc_rays(const double* rec, int64_t n_gen, int d, double sqmax,
               const vr_screen32* s32, const double* cand_rec, const int32_t* cand, int64_t n_cand,
               const int32_t* cells, int64_t n_cells, int64_t rays_per_cell,
               const double* dirs, uint64_t seed,
               int32_t* out_idx, double* out_t, uint8_t* out_flag,
               int32_t* recheck_list, int32_t* recheck_count, void* stream);

/* vr_mc_rays through the pruned index (rays of one cell are coherent). */
int vr_mc_rays_pruned(const double* rec, int64_t n_gen, int d, double sqmax,
                      const vr_screen32* s32, const vr_prune_index* ix, const int32_t* cells,
                      int64_t n_cells, int64_t rays_per_cell, const double* dirs,
                      uint64_t seed, const int32_t* order, int32_t* out_idx,
                      double* out_t, uint8_t* out_flag, int32_t* recheck_list,
                      int32_t* recheck_count, uint64_t* work, void* stream);

int vr_mc_recheck(const double* rec, int64_t n_gen, int d,
                  const double* cand_rec, const int32_t* cand, int64_t n_cand,
                  const int32_t* cells, int64_t rays_per_cell,
                  const double* dirs, uint64_t seed,
                  const int32_t* recheck_list, const int32_t* recheck_count,
                  int64_t max_list, int32_t* out_idx, double* out_t,
                  uint8_t* out_flag, void* stream);

int64_t vr_mc_map_bytes(int64_t n_blocks, int max_faces, int integrate);
int vr_mc_reduce(const double* rec, int d, const int32_t* cells,
                 int64_t n_cells, int64_t rays_per_cell, const double* dirs,
                 uint64_t seed, const int32_t* ray_idx, const double* ray_t,
                 const uint8_t* ray_flag, int max_faces,
                 int degenerate_is_error, double surf,
                 const int32_t* cell_sel, int64_t n_sel, void* map_ws, int64_t map_ws_bytes,
                 double* out_volume, int32_t* out_face_j, double* out_face_area,
                 int32_t* out_nfaces, int32_t* out_status,
                 int64_t* out_first_bad, double* out_samples /* nullable */,
                 void* stream);

/* MC with an integrand (reference mc_integrate_cell, integrate_mc.py:70-121):
 * as vr_mc_reduce (degenerate rays always count), plus per-face surface
 * integrals sum_rays f(rp) w and the volume integral
 * sum_rays [sum_{s<m} f(x_c + t_s seg) t_s^(d-1)] length^d, scaled like the
 * reference.  integrand_kind: 1 const (coef[0]), 2 sin(x_1^2), 3 linear
 * (coef[0..d-1] . x + coef[d]) -- the reference's built-ins
 * (integrands.py:10-44); `coef` is a HOST array (copied into the launch).  Subsample positions t_s come from `unif`
 * ((n_rays, m) replayed uniforms) or, when NULL, from Philox counter
 * (ray, cell, 0x100 + s/2, 'MU') keyed by `seed`. */
int vr_mc_integrate(const double* rec, int d, const int32_t* cells, int64_t n_cells,
                    int64_t rays_per_cell, const double* dirs, uint64_t seed,
                    const int32_t* ray_idx, const double* ray_t,
                    const uint8_t* ray_flag, int max_faces, double surf,
                    int integrand_kind, const double* coef, int m_sub,
                    const double* unif, const int32_t* cell_sel, int64_t n_sel,
                    void* map_ws, int64_t map_ws_bytes, double* out_volume, int32_t* out_face_j,
                    double* out_face_area, double* out_face_surf,
                    double* out_vol_integral, int32_t* out_nfaces,
                    int32_t* out_status, int64_t* out_first_bad, void* stream);

/* The Philox subsample uniforms of vr_mc_integrate, (n, m) fp64. */
int vr_mc_uniforms(int64_t n_cells, const int32_t* cells, int64_t rays_per_cell,
                   int m_sub, uint64_t seed, double* out_u, void* stream);

/* Export the unit directions the Philox path uses (for RNG replay into the
 * reference, SURVEY.md §8(c) rule 4): raw Gaussian draws z, (n, d) fp64. */
int vr_mc_directions(int d, int64_t n_cells, const int32_t* cells,
                     int64_t rays_per_cell, uint64_t seed, double* out_z,
                     void* stream);

/* ---- Level-synchronous traversal (reference voronoi_graph DFS,
 *      graph.py:88-146, reformulated per SURVEY.md §7 K2) -------------------
 * Device hash tables, open-addressed with linear probing; capacities are
 * powers of two; slot state 0 empty / 1 being written / 2 published. */
typedef struct vr_traverse_tables {
  int32_t* vkeys;   /* vcap * (d+1) sorted sigma keys                        */
  int32_t* vstate;  /* vcap                                                  */
  int32_t* vval;    /* vcap: vertex id (or smallest claiming ray this level) */
  int32_t* vlevel;  /* vcap: level at which the key was inserted             */
  int64_t vcap;
  int32_t* ekeys;   /* ecap * d sorted eta keys                              */
  int32_t* estate;  /* ecap                                                  */
  int32_t* ecount;  /* ecap: number of discovered incident vertices.  The two
                       arrays may be ONE array of 2 * ecap int32 holding
                       (state, count) pairs -- pass ecount == estate + 1 -- so
                       that a slot's state and counter share a 32-B sector (one
                       random sector less per bump); every vr_trav_* call taking
                       the tables (and the old-table arguments of
                       vr_trav_rehash_edges) recognises the pair layout by that
                       pointer relation.  vr_trav_published reads a plain state
                       array (stride 1) only.                                */
  int64_t ecap;
  int32_t* overflow;/* 1 int32: set when a probe sequence exhausts a table   */
} vr_traverse_tables;

/* Native level driver (csrc/level.cu): one traversal level in two calls,
 * each ending with a stream synchronisation.
 * vr_trav_level_open: open edges of the n_v frontier vertices (as
 *   vr_trav_open_edges), their exclusive int64 offsets in open_off, and the
 *   ray count R in *n_rays_out (host).
 * vr_trav_level_cast: the R edge rays (as vr_trav_emit_rays; bad[0..1] are
 *   zeroed first), their processing order (vr_ray_order), the pruned RayCast with |eta| = d plus the exact re-check (hits in
 *   hit_idx / hit_t / hit_flag), vr_trav_claim, exclusive offsets of the new
 *   vertices and of the escapes, and counts_out[5] (host) = {new vertices,
 *   escapes, degenerate rays, affinely dependent frontier vertices, table
 *   overflow}.  Requires the pruned index (n_gen >= 256 in the Python API);
 *   the caller then grows the edge table if needed and runs
 *   vr_trav_finalize / vr_trav_boundary. */
int vr_trav_level_open(const vr_traverse_tables* tab, int d, const int32_t* frontier_sigma,
                       int64_t n_v, uint8_t* open_mask, int32_t* open_count, int64_t* open_off,
                       int64_t* n_rays_out, void* workspace, int64_t workspace_bytes,
                       void* stream);
int vr_trav_level_cast(const vr_traverse_tables* tab, const double* rec, int64_t n_gen, int d,
                       double sqmax, const vr_screen32* s32, const vr_prune_index* ix,
                       const int32_t* frontier_sigma, const double* frontier_r, int64_t n_v,
                       const uint8_t* open_mask, const int64_t* open_off, int64_t n_rays,
                       int32_t level, double* ray_x, double* ray_u, int32_t* ray_eta,
                       int32_t* ray_parent, int32_t* hit_idx, double* hit_t, uint8_t* hit_flag,
                       int32_t* ray_sigma, int64_t* slot, int32_t* new_flag, int32_t* esc_flag,
                       int64_t* new_off, int64_t* esc_off, int32_t* bad, uint64_t* work,
                       int64_t* counts_out, void* workspace, int64_t workspace_bytes,
                       void* stream);
/* Device scratch (bytes) both calls need for n_v frontier vertices and
 * n_rays edge rays (n_rays = 0: vr_trav_level_open only); a smaller
 * workspace returns VR_ECAPACITY. */
int vr_trav_level_workspace(int64_t n_v, int64_t n_rays, int64_t n_gen, int d, int64_t* bytes);

/* Native multi-level driver: the whole level loop in C++ (open -> capacity
 * checks -> cast -> finalize + boundary per level, the two synchronisations
 * of the level calls and no other host work).  Runs levels state->level ..
 * last_level (-1: until no vertex is new) over the frontier [f0, f1) of
 * vertex ids; level_new[l] receives the new-vertex count of level l.  It
 * returns VR_OK with state->need = VR_RUN_DONE, or with a capacity the
 * caller must grow (workspace bytes, vertex arrays / table, edge table,
 * boundary arrays: need_amount) before calling again -- state->phase
 * remembers a level whose cast is done -- or VR_RUN_ERROR with the
 * degenerate / affinely dependent / overflow counts set.  Workspace size for
 * F frontier vertices and R rays: vr_trav_run_workspace. */
enum vr_run_need {
  VR_RUN_DONE = 0,
  VR_RUN_NEED_WORKSPACE = 1,
  VR_RUN_NEED_VERTICES = 2,
  VR_RUN_NEED_EDGES = 3,
  VR_RUN_NEED_BOUNDARY = 4,
  VR_RUN_ERROR = 5
};
typedef struct vr_trav_state {
  int32_t* vsig;         /* vertex arrays: sigma (vcap_arrays, d+1), r (vcap_arrays, d) */
  double* vr;
  int64_t vcap_arrays;
  int32_t* bsig;         /* boundary rays: sigma (bcap, d+1), u (bcap, d) */
  double* bu;
  int64_t bcap;
  int64_t nv, nb, e_ub;  /* vertices, boundary rays, edge incidences so far */
  int64_t f0, f1;        /* frontier: vertex ids [f0, f1) */
  int32_t level;         /* level to run next */
  int32_t phase;         /* 0: level not started, 2: open step done (its result is
                            the workspace prefix: grow the workspace keeping its
                            contents), 1: cast done, finalize pending */
  int64_t pending_rays;
  int64_t n_new, n_esc, n_degenerate, n_bad, overflow;  /* last cast */
  int64_t rays;          /* edge raycasts so far */
  int32_t need;          /* vr_run_need */
  int64_t need_amount;
  int32_t sub_n, sub_j;  /* sub-rounds of the current level (set by the driver;
                            start at 0): round sub_j of sub_n is next */
} vr_trav_state;
int vr_trav_run_workspace(int64_t n_frontier, int64_t n_rays, int64_t n_gen, int d,
                          int64_t* bytes);
/* Sub-rounds of large levels in vr_trav_run: a level of F frontier vertices is
 * cast in about F (d + 1) / 2 / rays_per_round interleaved rounds (at most
 * max_rounds <= 64; vertex v of the frontier belongs to round v % rounds), so
 * that vertices found by an earlier round close the edges later rounds would
 * have cast (graph.py:115-128).  rays_per_round 0 = never split; -1 / -1 =
 * back to the defaults (environment VR_SUB_RAYS / VR_SUB_MAX).  The vertex
 * set, edge counts and boundary rays do not depend on the setting; vertex ids
 * within a level do.  Process-wide. */
int vr_trav_set_sub_rounds(int64_t rays_per_round, int max_rounds);
int vr_trav_run(const vr_traverse_tables* tab, vr_trav_state* state, const double* rec,
                int64_t n_gen, int d, double sqmax, const vr_screen32* s32,
                const vr_prune_index* ix, int32_t last_level, int64_t* level_new,
                int64_t level_cap, uint64_t* work, void* workspace, int64_t workspace_bytes,
                void* stream);

/* Register vertices (sigma (n_v, d+1) sorted) with ids base_id.. at `level`;
 * optionally bump the counters of their d+1 edges (graph.py:115-120). */
int vr_trav_insert_vertices(const vr_traverse_tables* tab, int d,
                            const int32_t* sigma, int64_t n_v, int32_t base_id,
                            int32_t level, int bump_edges, void* stream);

/* Re-insert the published slots of an old edge table into tab (growth). */
int vr_trav_rehash_edges(const vr_traverse_tables* tab, int d,
                         const int32_t* okeys, const int32_t* ostate,
                         const int32_t* ocount, int64_t ocap, void* stream);

/* vr_trav_open_edges restricted to the frontier vertices with
 * v % sub_n == sub_j (sub-rounds of a level; the others report no open edge). */
int vr_trav_open_edges_sub(const vr_traverse_tables* tab, int d,
                           const int32_t* sigma, int64_t n_v, int sub_n, int sub_j,
                           uint8_t* open_mask, int32_t* open_count, void* stream);

/* open_mask[v*(d+1)+k] = 1 iff edge sigma_v \ sigma_v[k] has count < 2
 * (graph.py:127-128); open_count[v] = number of open edges of v. */
int vr_trav_open_edges(const vr_traverse_tables* tab, int d,
                       const int32_t* sigma, int64_t n_v, uint8_t* open_mask,
                       int32_t* open_count, void* stream);

/* One ray per open edge at exclusive offset open_off[v] (+ rank among v's
 * open edges): x = r_v, u = outward direction (raycast.py:345-378),
 * eta = sigma_v \ sigma_v[k], parent = v.  *bad counts singular simplices. */
int vr_trav_emit_rays(const double* rec, int d, const int32_t* sigma,
                      const double* r, int64_t n_v, const uint8_t* open_mask,
                      const int64_t* open_off, double* ray_x, double* ray_u,
                      int32_t* ray_eta, int32_t* ray_parent, int32_t* bad,
                      void* stream);

/* sigma' = sorted(eta + {hit}) per hit ray; insert-or-find in the vertex
 * table; the smallest ray id claims each key first seen at `level`.
 * new_flag[k] = 1 for the claiming ray, esc_flag[k] = 1 for escaped rays. */
int vr_trav_claim(const vr_traverse_tables* tab, int d, const int32_t* ray_eta,
                  const int32_t* hit_idx, const uint8_t* hit_flag,
                  int64_t n_rays, int32_t level, int32_t* out_sigma,
                  int64_t* out_slot, int32_t* new_flag, int32_t* esc_flag,
                  void* stream);

/* New vertex base_id + new_off[k]: store sigma', its fp64 circumcentre
 * (no chained drift, SURVEY.md §8(c) rule 3) and, with bump != 0, bump its
 * edge counters (graph.py:115-120; the owner-sharded traversal bumps at
 * the edge owners instead, vr_trav_bump_keys). */
int vr_trav_finalize(const vr_traverse_tables* tab, const double* rec, int d,
                     const int32_t* ray_sigma, const int64_t* slot,
                     const int32_t* new_flag, const int64_t* new_off,
                     int64_t n_rays, int32_t base_id, int32_t* vsig, double* vr,
                     int32_t* bad, int bump, void* stream);

/* ---- Owner-sharded traversal (csrc/shard.cu) -------------
 * Vertex sigma lives on rank owner(sigma), edge eta on owner(eta) (a hash of
 * the sorted tuple, high bits, mod n_parts).  Per level each rank raycasts
 * the open edges of its own frontier (vr_shard_open: open iff the edge's
 * count, returned by its owner at the previous level, is < 2 --
 * graph.py:127-128; vr_trav_level_rays: rays + order + pruned RayCast +
 * exact re-check), sends the hit sigma' to their owners (vr_shard_bucket +
 * an all-to-all), which dedupe them (vr_trav_claim_sigma: insert-or-find,
 * smallest received row wins) and store the new vertices
 * (vr_trav_finalize, bump = 0); the new vertices' edges (vr_vertex_edges)
 * go to the edge owners, which bump them and answer with the counts
 * (vr_trav_bump_keys) -- the next level's open test.  Results are those of
 * the single-GPU level-synchronous traversal for any rank count.
 *
 * vr_shard_bucket: owner of each of n rows of k int32, a stable send order
 *   perm (grouped by owner) and per-owner counts (device int64[n_parts]).
 * vr_shard_gather_rows: out[i] = rows[perm[i]]; vr_shard_scatter_rows:
 *   out[perm[i]] = rows[i] (k int32 per row).
 * vr_shard_open: open mask / counts / exclusive offsets from per-vertex edge
 *   counts (n_v, d+1), the ray count in *n_rays_out (host, synchronises). */
int vr_shard_bucket(const int32_t* rows, int64_t n, int k, int n_parts, int32_t* perm,
                    int64_t* counts, void* workspace, int64_t* workspace_bytes, void* stream);
int vr_shard_gather_rows(const int32_t* rows, int k, const int32_t* perm, int64_t n,
                         int32_t* out, void* stream);
int vr_shard_scatter_rows(const int32_t* rows, int k, const int32_t* perm, int64_t n,
                          int32_t* out, void* stream);
int vr_shard_open(const int32_t* edge_counts, int64_t n_v, int d, uint8_t* open_mask,
                  int32_t* open_count, int64_t* open_off, int64_t* n_rays_out, void* workspace,
                  int64_t* workspace_bytes, void* stream);
int vr_trav_claim_sigma(const vr_traverse_tables* tab, int d, const int32_t* rows, int64_t n,
                        int32_t level, int64_t* out_slot, int32_t* new_flag, void* stream);
int vr_trav_bump_keys(const vr_traverse_tables* tab, int d, const int32_t* keys, int64_t n,
                      int32_t* counts_out, void* stream);
/* The d+1 edges (d-subsets, sigma[k] omitted, k = 0..d) of n_v sigma rows. */
int vr_vertex_edges(const int32_t* sigma, int64_t n_v, int d, int32_t* out, void* stream);
/* vr_trav_level_cast without the local claim: the R edge rays of the
 * frontier (emit), their order, the pruned RayCast + re-check; counts_out[3]
 * (host) = {escapes, degenerate rays, affinely dependent frontier vertices}.
 * Workspace: vr_trav_level_workspace(n_v, n_rays, ...). */
int vr_trav_level_rays(const double* rec, int64_t n_gen, int d, double sqmax,
                       const vr_screen32* s32, const vr_prune_index* ix,
                       const int32_t* frontier_sigma, const double* frontier_r, int64_t n_v,
                       const uint8_t* open_mask, const int64_t* open_off, int64_t n_rays,
                       double* ray_x, double* ray_u, int32_t* ray_eta, int32_t* ray_parent,
                       int32_t* hit_idx, double* hit_t, uint8_t* hit_flag, int32_t* bad,
                       uint64_t* work, int64_t* counts_out, void* workspace,
                       int64_t workspace_bytes, void* stream);

/* Escaped rays -> BoundaryRay(sigma_parent, u) at base_b + esc_off[k]
 * (graph.py:138-139). */
int vr_trav_boundary(int d, const int32_t* esc_flag, const int64_t* esc_off,
                     const int32_t* ray_parent, const double* ray_u,
                     int64_t n_rays, const int32_t* frontier_sigma,
                     int64_t base_b, int32_t* bsig, double* bu, void* stream);

/* flag[h] = (state[h] == 2), for compaction of a table. */
int vr_trav_published(const int32_t* state, int64_t cap, int32_t* flag,
                      void* stream);

/* Edge-table compaction in two passes (slot order, the same order as
 * vr_trav_published + prefix sum + vr_trav_edge_compact):
 * vr_trav_edges_count: published slots per chunk of 4096, exclusive offsets
 *   in chunk_off (ceil(ecap / 4096) + 1 int64; the last entry is the total),
 *   *n_edges (host) = the total; ends with a stream synchronisation.  NULL
 *   workspace: *workspace_bytes = the scan scratch needed.
 * vr_trav_edges_compact: the slot of every published row (out_slot,
 *   n_edges int64 scratch), then keys (n_edges, d) and counts in slot
 *   order. */
int vr_trav_edges_count(const vr_traverse_tables* tab, int64_t* chunk_off,
                        int64_t* n_edges, void* workspace, int64_t* workspace_bytes,
                        void* stream);
int vr_trav_edges_compact(const vr_traverse_tables* tab, int d,
                          const int64_t* chunk_off, int64_t n_edges, int64_t* out_slot,
                          int32_t* out_keys, int32_t* out_count, void* stream);

/* Compact the edge table (published slots, exclusive offsets `off`). */
int vr_trav_edge_compact(const vr_traverse_tables* tab, int d,
                         const int64_t* off, int32_t* out_keys,
                         int32_t* out_count, void* stream);

/* ---- Host descent streams (host code; no GPU needed) ----------------------
 * stream(seed, tag, index) of the reference (pkg/src/voronray/rng.py:18-28):
 * numpy Generator(PCG64(SeedSequence(entropy=seed, spawn_key=(tag, index)))),
 * restated over arrays of streams.  vr_host_streams writes 4 uint64 per
 * stream (PCG64 state high, low, increment high, low); vr_host_normals draws
 * `count` standard normals per listed stream (rows[i], or i when rows is
 * NULL) into out[i * count ..] with NumPy's ziggurat (libnpyrandom, linked
 * in) and advances the states: bit-identical to
 * Generator.standard_normal(count) (descent, graph.py:46-85). */
int vr_host_streams(uint64_t seed, uint64_t tag, const int64_t* index, int64_t n,
                    uint64_t* state);
int vr_host_normals(uint64_t* state, const int64_t* rows, int64_t n, int64_t count,
                    double* out);

/* Roofline probe: `blocks` x 256 threads x iters x 8 independent FMA chains
 * (dtype 0 = fp64 DFMA, 1 = fp32 FFMA; flops = 4096 * iters * blocks) or
 * 8 independent tf32 mma.sync m16n8k8 per warp (dtype 2, the legacy warp
 * tensor path of the pruned kernel's screen; flops = 131072 * iters * blocks).
 * Used by bench.py to measure the FP64 / FP32 / warp-MMA peaks live
 * (MEASURED_PEAKS.json has only HBM and bf16). */
int vr_fma_probe(int dtype, int blocks, int iters, void* scratch, void* stream);

/* ---- HMC post-processing --------------------------
 * Replaces integrate_hmc.py:21-91 (hmc_volume, hmc_interface_integral,
 * hmc_cell_integral) with segmented reductions over the sigma-keyed vertex
 * set.
 *
 * vr_hmc_face_index: the interface index of a mesh (sigma (n_v, d+1) sorted
 *   rows, edges (n_e, d) with counts): keys / vid (n_v d(d+1)/2 each) = the
 *   (generator pair, vertex id) incidences radix-sorted by pair (stable, so
 *   an interface's vertices stay in vertex order: Mesh.face_vertices,
 *   core.py:223-246); ukeys (<= n_e d(d-1)/2) = sorted generator pairs of the
 *   boundary edges (count 1: Mesh.face_is_unbounded, core.py:262-276),
 *   *n_ukeys_out (host; the call synchronises); cell_unbounded (n_gen uint8:
 *   Mesh.unbounded_cells); nb_count (n_gen int32: |Mesh.neighbors(i)|).
 *   workspace == NULL: *workspace_bytes receives the scratch size.
 * vr_hmc_faces: per queried interface (face_i, face_j, area): the vertex run
 *   [out_first, + out_count) in `vid`, status (0 ok, 1 unbounded interface,
 *   2 fewer than d vertices -- the reference raises UnboundedFace for both --
 *   3 not an interface of the mesh), the vertex mean of f (compensated sum;
 *   the reference uses math.fsum), the vertex centroid and
 *   F = (d mean + f(centroid)) A / (d + 1) (integrate_hmc.py:42-64).
 *   integrand_kind 0 skips f (centroid / counts only), else 1 const, 2
 *   sin(x_1^2), 3 linear (integrands.py:10-44); coef is a HOST array.
 * vr_hmc_cells: per cell c with faces [face_off[c], face_off[c+1]):
 *   volume = (1/d) sum_j |x_i - x_j|/2 A_ij (integrate_hmc.py:21-39) and,
 *   with an integrand, (d sum_j h_j F_ij / d + f(x_i) V) / (d + 1)
 *   (integrate_hmc.py:67-91; V = volume_in[c] when given, else the pyramid
 *   volume); out_status bit 0 unbounded cell (UnboundedCell), bit 1 a mesh
 *   neighbour without an area (MissingNeighbor), bit 2 a failed interface. */
int vr_hmc_face_index(const int32_t* sigma, int64_t n_v, int d, int64_t n_gen,
                      const int32_t* edge_key, const int32_t* edge_count, int64_t n_e,
                      uint64_t* keys, int32_t* vid, uint64_t* ukeys, int64_t* n_ukeys_out,
                      uint8_t* cell_unbounded, int32_t* nb_count, void* workspace,
                      int64_t* workspace_bytes, void* stream);
int vr_hmc_faces(const uint64_t* keys, const int32_t* vid, int64_t n_keys, const uint64_t* ukeys,
                 int64_t n_ukeys, const double* r, int d, const int32_t* face_i,
                 const int32_t* face_j, const double* area, int64_t n_f, int integrand_kind,
                 const double* coef, double* out_F, int32_t* out_status, int32_t* out_first,
                 int32_t* out_count, double* out_mean, double* out_centroid, void* stream);
int vr_hmc_cells(const double* rec, int d, const int32_t* cells, int64_t n_c,
                 const int64_t* face_off, const int32_t* face_j, const double* area,
                 const double* F, const int32_t* face_status, const uint8_t* cell_unbounded,
                 const int32_t* nb_count, int integrand_kind, const double* coef,
                 const double* volume_in, double* out_volume, double* out_integral,
                 int32_t* out_status, void* stream);

/* ---- Mesh arrays (csrc/mesh.cu) ------------------------------------------
 * vr_lex_order: stable lexicographic order of n rows of k int32 (k LSD
 *   radix passes), order[i] = row id -- the order of `sorted()` over sigma /
 *   eta tuples (the reference's dict views, core.py:205-221).
 * vr_edge_incidence: the d-subsets of the n_v sigma rows (every vertex is
 *   incident to its d+1 edges, graph.py:115-120) as distinct lexicographically
 *   sorted keys (out_keys, <= n_v (d+1) rows of d) with their incidence
 *   counts; *n_unique_out (host; the call synchronises).
 * vr_edge_check: incident[e] = incidence count of recorded edge e (0 if no
 *   vertex has it) -- verify_mesh's edge-consistency pass (graph.py:214-229).
 * Workspace convention as vr_ray_order (NULL: size query). */
int vr_lex_order(const int32_t* rows, int64_t n, int k, int32_t* order, void* workspace,
                 int64_t* workspace_bytes, void* stream);
int vr_edge_incidence(const int32_t* sigma, int64_t n_v, int d, int32_t* out_keys,
                      int32_t* out_counts, int64_t* n_unique_out, void* workspace,
                      int64_t* workspace_bytes, void* stream);
int vr_edge_check(const int32_t* inc_keys, const int32_t* inc_counts, int64_t n_inc,
                  const int32_t* edge_keys, int64_t n_e, int d, int32_t* incident, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VORONRAY_B200_H */
