// Native build of the pruned RayCast's kd index (vr_prune_index), the fp32
// screening frame (vr_screen32_stats) and the processing order of a ray batch
// (vr_ray_keys / vr_ray_order).
//
// The reference pays for its spatial index inside NodeSet.__init__
// (pkg/src/voronray/core.py:52-57, scipy cKDTree over the generators); this is
// the B200 counterpart.  The index is a balanced kd partition of the
// generators into tiles of VR_PRUNE_TILE records, built level by level:
//
//   depth l:  every heap node at depth l that covers > 1 tile takes the
//             bounding box of its current elements (warp reduction +
//             order-preserving integer atomics), picks the widest axis (first
//             on ties), and its elements are stably sorted along that axis
//             (cub radix sort of the fp64 coordinate, then a stable radix sort
//             by segment so every node keeps its position range); the node
//             splits after floor(tiles / 2) whole tiles.
//
// A node covering tiles [lo, hi) splits at lo + (hi - lo) / 2, so the heap
// ranges are known before any element moves (k_node_ranges); only the order
// inside the ranges is computed.  Then the kd-ordered records are gathered,
// and tile / node / 32-ary boxes (fp64 and outward-rounded fp32 in the
// centred frame) and the fp32 / tensor-core screening copies are packed.
// Everything lives in one caller-owned arena; scratch comes from a caller
// workspace (include/voronray_b200.h: nothing persistent is allocated).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

extern "C" {
int vr_pack_records32(const double* rec, int64_t rows, int d, const double* center,
                      float* rec32, void* stream);
int vr_pack_records32_pairs(const float* rec32, int64_t rows, int d, float* out, void* stream);
int vr_pack_records_mma(const float* rec32, int64_t rows, int d, float* out, void* stream);
int vr_pack_records_umma(const float* rec32, int64_t rows, int d, float* out, void* stream);
}

namespace {

constexpr int TILE = VR_PRUNE_TILE;
constexpr int WIDE = 32;

__host__ __device__ constexpr int box32_stride(int d) { return (2 * d + 3) & ~3; }

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline unsigned grid_for(int64_t n, int nt = 256, int64_t cap = 8192) {
  int64_t b = (n + nt - 1) / nt;
  if (b < 1) b = 1;
  return (unsigned)(b < cap ? b : cap);
}

// Order-preserving map fp64 -> uint64 (for atomicMin / atomicMax).
__device__ __forceinline__ unsigned long long enc_d(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dec_d(unsigned long long e) {
  const unsigned long long b = (e >> 63) ? (e & 0x7fffffffffffffffull) : ~e;
  return __longlong_as_double((long long)b);
}

// Heap node i covers tiles [lo, hi) of nt; false if the slot is unused.
__device__ __forceinline__ bool heap_range(int64_t i, int64_t nt, int64_t& lo, int64_t& hi) {
  const unsigned long long v = (unsigned long long)i + 1;
  const int depth = 63 - __clzll(v);
  lo = 0;
  hi = nt;
  for (int b = depth - 1; b >= 0; --b) {
    const int64_t n = hi - lo;
    if (n <= 1) return false;
    const int64_t mid = lo + n / 2;
    if ((v >> b) & 1ull) lo = mid; else hi = mid;
  }
  return true;
}

// The node at depth `depth` on tile t's root path (heap index), or the leaf
// above it if t's leaf is shallower (then *at_depth = false).
__device__ __forceinline__ int64_t node_at_depth(int64_t t, int64_t nt, int depth, int64_t& lo,
                                                 int64_t& hi, bool& at_depth) {
  lo = 0;
  hi = nt;
  int64_t node = 0;
  for (int s = 0; s < depth; ++s) {
    const int64_t n = hi - lo;
    if (n <= 1) {
      at_depth = false;
      return node;
    }
    const int64_t mid = lo + n / 2;
    if (t < mid) { hi = mid; node = 2 * node + 1; }
    else { lo = mid; node = 2 * node + 2; }
  }
  at_depth = true;
  return node;
}

__global__ void k_node_ranges(int64_t nn, int64_t nt, int32_t* __restrict__ range) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo, hi;
    const bool ok = heap_range(i, nt, lo, hi);
    range[2 * i] = ok ? (int32_t)lo : -1;
    range[2 * i + 1] = ok ? (int32_t)hi : -1;
  }
}

__global__ void k_iota32(int32_t* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

__global__ void k_fill_u64(unsigned long long* __restrict__ v, int64_t n, unsigned long long a,
                           unsigned long long b) {
  // even entries a, odd entries b
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (i & 1) ? b : a;
}

// Bounding boxes of the splitting nodes at `depth` over their current
// elements.  Tiles are 64 rows, so the 32 positions of an aligned warp share
// one tile (and one node): a warp reduction, then 2d atomics by lane 0.
// bbox[(node - first) * 2d + 2k] = enc(min_k), [.. + 2k + 1] = enc(max_k).
template <int D>
__global__ void k_level_bbox(const double* __restrict__ rec, const int32_t* __restrict__ order,
                             int64_t n, int64_t nt, int depth,
                             unsigned long long* __restrict__ bbox) {
  constexpr int S = rec_stride(D);
  const int lane = threadIdx.x & 31;
  const int64_t first = ((int64_t)1 << depth) - 1;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = base + lane;
    int64_t lo, hi;
    bool at;
    const int64_t node = node_at_depth(base / TILE, nt, depth, lo, hi, at);
    if (!at || hi - lo <= 1) continue;  // warp-uniform
    double mn[D], mx[D];
    if (p < n) {
      const double* x = rec + (int64_t)order[p] * S;
#pragma unroll
      for (int k = 0; k < D; ++k) mn[k] = mx[k] = x[k];
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) { mn[k] = CUDART_INF; mx[k] = -CUDART_INF; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
        mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
      }
    }
    if (lane == 0) {
      unsigned long long* b = bbox + (node - first) * 2 * D;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        atomicMin(b + 2 * k, enc_d(mn[k]));
        atomicMax(b + 2 * k + 1, enc_d(mx[k]));
      }
    }
  }
}

// Sort keys of one level: the coordinate along the node's widest axis (0
// for elements whose node does not split: the stable sorts keep their
// order), and as value the element id packed with its segment key (first
// tile of the node that holds it at this depth).
template <int D>
__global__ void k_level_keys(const double* __restrict__ rec, const int32_t* __restrict__ order,
                             int64_t n, int64_t nt, int depth,
                             const unsigned long long* __restrict__ bbox,
                             double* __restrict__ key, unsigned long long* __restrict__ val) {
  constexpr int S = rec_stride(D);
  const int64_t first = ((int64_t)1 << depth) - 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo, hi;
    bool at;
    const int64_t node = node_at_depth(p / TILE, nt, depth, lo, hi, at);
    const int32_t id = order[p];
    double kv = 0.0;
    if (at && hi - lo > 1) {
      const unsigned long long* b = bbox + (node - first) * 2 * D;
      int dim = 0;
      double best = -1.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double ext = dec_d(b[2 * k + 1]) - dec_d(b[2 * k]);
        if (ext > best) { best = ext; dim = k; }  // first axis on ties
      }
      kv = rec[(int64_t)id * S + dim];
    }
    key[p] = kv;
    val[p] = ((unsigned long long)(uint32_t)lo << 32) | (uint32_t)id;
  }
}

__global__ void k_split_val(const unsigned long long* __restrict__ val, int64_t n,
                            uint32_t* __restrict__ seg, int32_t* __restrict__ id) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = val[p];
    seg[p] = (uint32_t)(v >> 32);
    id[p] = (int32_t)(uint32_t)v;
  }
}

// kd-ordered records (sentinel rows past n), perm, inv_perm.
template <int D>
__global__ void k_gather(const double* __restrict__ rec, const int32_t* __restrict__ order,
                         int64_t n, int64_t rows, double* __restrict__ crec,
                         int32_t* __restrict__ perm, int32_t* __restrict__ inv_perm) {
  constexpr int S = rec_stride(D);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < rows;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (p < n) {
      const int32_t id = order[p];
      perm[p] = id;
      inv_perm[id] = (int32_t)p;
#pragma unroll
      for (int k = 0; k < S; ++k) crec[p * S + k] = rec[(int64_t)id * S + k];
    } else {
#pragma unroll
      for (int k = 0; k < S; ++k) crec[p * S + k] = (k == D) ? CUDART_INF : 0.0;
    }
  }
}

// fp64 box of each tile (one warp per tile, <= 64 valid rows).
template <int D>
__global__ void k_tile_box(const double* __restrict__ crec, int64_t n, int64_t nt,
                           double* __restrict__ tile_box) {
  constexpr int S = rec_stride(D);
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < nt;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double mn[D], mx[D];
#pragma unroll
    for (int k = 0; k < D; ++k) { mn[k] = CUDART_INF; mx[k] = -CUDART_INF; }
    for (int r = lane; r < TILE; r += 32) {
      const int64_t p = t * TILE + r;
      if (p < n) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const double v = crec[p * S + k];
          mn[k] = fmin(mn[k], v);
          mx[k] = fmax(mx[k], v);
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
        mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
      }
    }
    if (lane < D) {
      double a = mn[0], b = mx[0];
#pragma unroll
      for (int k = 1; k < D; ++k) if (lane == k) { a = mn[k]; b = mx[k]; }
      tile_box[t * 2 * D + lane] = a;
      tile_box[t * 2 * D + D + lane] = b;
    }
  }
}

// Union of the tile boxes [t0, t1) (one warp); fp64 [lo.., hi..] into out.
template <int D>
__device__ void union_tiles(const double* __restrict__ tile_box, int64_t t0, int64_t t1,
                            double* __restrict__ out, int lane) {
  double mn[D], mx[D];
#pragma unroll
  for (int k = 0; k < D; ++k) { mn[k] = CUDART_INF; mx[k] = -CUDART_INF; }
  for (int64_t t = t0 + lane; t < t1; t += 32) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      mn[k] = fmin(mn[k], tile_box[t * 2 * D + k]);
      mx[k] = fmax(mx[k], tile_box[t * 2 * D + D + k]);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
      mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) { out[k] = mn[k]; out[D + k] = mx[k]; }
  }
}

// fp32 row of one fp64 box in the frame centred at c: outward [lo, hi]
// (lo rounded down, hi rounded up) and centre / half-extent [c, h] with
// [c - h, c + h] containing the box (h rounded up).
template <int D>
__device__ void box32_rows(const double* __restrict__ box, const double* __restrict__ c,
                           float* __restrict__ out_lohi, float* __restrict__ out_ch) {
  constexpr int B32 = box32_stride(D);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const double lo = box[k] - c[k], hi = box[D + k] - c[k];
    if (out_lohi) {
      out_lohi[k] = __double2float_rd(lo);
      out_lohi[D + k] = __double2float_ru(hi);
    }
    if (out_ch) {
      const float c32 = __double2float_rn(0.5 * (lo + hi));
      const double c64 = (double)c32;
      const double h = fmax(hi - c64, c64 - lo);
      out_ch[k] = c32;
      out_ch[D + k] = __double2float_ru(h);
    }
  }
#pragma unroll
  for (int k = 2 * D; k < B32; ++k) {
    if (out_lohi) out_lohi[k] = 0.0f;
    if (out_ch) out_ch[k] = 0.0f;
  }
}

template <int D>
__global__ void k_tile_box32(const double* __restrict__ tile_box, int64_t nt,
                             const double* __restrict__ c, float* __restrict__ tile_box32) {
  constexpr int B32 = box32_stride(D);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x)
    box32_rows<D>(tile_box + t * 2 * D, c, tile_box32 + t * B32, nullptr);
}

// Node boxes: the union of the node's tile range; unused heap slots get a
// finite all-zero box (never visited).
template <int D>
__global__ void k_node_box(const double* __restrict__ tile_box, const int32_t* __restrict__ range,
                           int64_t nn, const double* __restrict__ c, double* __restrict__ node_box,
                           float* __restrict__ node_box32, float* __restrict__ node_cb32) {
  constexpr int B32 = box32_stride(D);
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < nn;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t lo = range[2 * i], hi = range[2 * i + 1];
    double* nb = node_box + i * 2 * D;
    if (lo < 0) {
      if (lane < 2 * D) nb[lane] = 0.0;
    } else {
      union_tiles<D>(tile_box, lo, hi, nb, lane);
    }
    __syncwarp();
    if (lane == 0) box32_rows<D>(nb, c, node_box32 + i * B32, node_cb32 + i * B32);
  }
}

// 32-ary tree over the tiles: level l node j = union of tiles
// [j 32^l, (j + 1) 32^l).  Rows of all levels back to back (wide_off).
template <int D>
__global__ void k_wide_box32(const double* __restrict__ tile_box, int64_t nt, int levels,
                             const int64_t* __restrict__ lvl_off_cnt,  // [off[8], cnt[8]] host-built
                             const double* __restrict__ c, float* __restrict__ wide32,
                             double* __restrict__ scratch) {
  constexpr int B32 = box32_stride(D);
  const int lane = threadIdx.x & 31;
  const int64_t total = lvl_off_cnt[levels - 1] + lvl_off_cnt[8 + levels - 1];
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < total;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int l = 0;
    while (l + 1 < levels && r >= lvl_off_cnt[l + 1]) ++l;
    const int64_t j = r - lvl_off_cnt[l];
    int64_t span = 1;
    for (int q = 0; q < l; ++q) span *= WIDE;
    const int64_t t0 = j * span;
    const int64_t t1 = (j + 1) * span < nt ? (j + 1) * span : nt;
    double* box = scratch + r * 2 * D;
    union_tiles<D>(tile_box, t0, t1, box, lane);
    __syncwarp();
    if (lane == 0) box32_rows<D>(box, c, wide32 + r * B32, nullptr);
  }
}

// Screening frame: centre = bounding-box midpoint (unless given), then
// max |x - c|^2 and max_k |x_k - c_k| (non-negative doubles order like their
// bit patterns).  stats layout: [0..7] centre, [8] sqmax, [9] bound,
// [16..31] encoded min / max (scratch).
template <int D>
__global__ void k_stats_minmax(const double* __restrict__ rec, int64_t n,
                               unsigned long long* __restrict__ mm) {
  constexpr int S = rec_stride(D);
  double mn[D], mx[D];
#pragma unroll
  for (int k = 0; k < D; ++k) { mn[k] = CUDART_INF; mx[k] = -CUDART_INF; }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double v = rec[i * S + k];
      mn[k] = fmin(mn[k], v);
      mx[k] = fmax(mx[k], v);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      mn[k] = fmin(mn[k], __shfl_xor_sync(0xffffffffu, mn[k], off));
      mx[k] = fmax(mx[k], __shfl_xor_sync(0xffffffffu, mx[k], off));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      atomicMin(mm + 2 * k, enc_d(mn[k]));
      atomicMax(mm + 2 * k + 1, enc_d(mx[k]));
    }
  }
}

template <int D>
__global__ void k_stats_centre(double* __restrict__ stats, const double* __restrict__ given) {
  const unsigned long long* mm = reinterpret_cast<const unsigned long long*>(stats + 16);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 8; ++k) {
      double c = 0.0;
      if (k < D) c = given ? given[k] : 0.5 * (dec_d(mm[2 * k]) + dec_d(mm[2 * k + 1]));
      stats[k] = c;
    }
    stats[8] = 0.0;
    stats[9] = 0.0;
  }
}

template <int D>
__global__ void k_stats_spread(const double* __restrict__ rec, int64_t n,
                               double* __restrict__ stats) {
  constexpr int S = rec_stride(D);
  double c[D];
#pragma unroll
  for (int k = 0; k < D; ++k) c[k] = stats[k];
  double sq = 0.0, bd = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double v = rec[i * S + k] - c[k];
      s += v * v;
      bd = fmax(bd, fabs(v));
    }
    sq = fmax(sq, s);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sq = fmax(sq, __shfl_xor_sync(0xffffffffu, sq, off));
    bd = fmax(bd, __shfl_xor_sync(0xffffffffu, bd, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(reinterpret_cast<unsigned long long*>(stats + 8),
              (unsigned long long)__double_as_longlong(sq));
    atomicMax(reinterpret_cast<unsigned long long*>(stats + 9),
              (unsigned long long)__double_as_longlong(bd));
  }
}

// Processing-order keys (key = base * 256 + direction class): base is the kd
// position of the ray's reference generator (inv_perm[eta[k * eta_len]]) or,
// with eta == NULL, k / per (MC: rays of one cell); the direction class is
// the signed index of the largest and second-largest |u_j| (< 256, d <= 8).
template <int D, typename K>
__global__ void k_ray_keys(const int32_t* __restrict__ inv_perm, const int32_t* __restrict__ eta,
                           int eta_len, int64_t per, const double* __restrict__ u, int64_t n,
                           K* __restrict__ keys, int32_t* __restrict__ iota) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double a1 = -1.0, a2 = -1.0;
    int i1 = 0, i2 = 0;
    bool s1 = false, s2 = false;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double v = u[k * D + j], a = fabs(v);
      if (a > a1) {  // first index on ties
        a2 = a1; i2 = i1; s2 = s1;
        a1 = a; i1 = j; s1 = v > 0.0;
      } else if (a > a2) {
        a2 = a; i2 = j; s2 = v > 0.0;
      }
    }
    const int64_t bucket = (int64_t)(i1 * 2 + (s1 ? 1 : 0)) * (2 * D) + (i2 * 2 + (s2 ? 1 : 0));
    const int64_t base = eta ? (int64_t)inv_perm[eta[k * eta_len]] : k / per;
    keys[k] = (K)(base * 256 + bucket);
    if (iota) iota[k] = (int32_t)k;
  }
}

int end_bit_for(int64_t max_key) {
  int b = 1;
  while (b < 63 && ((int64_t)1 << b) <= max_key) ++b;
  return b;
}

struct OrderPlan {
  bool narrow;
  int end_bit;
  size_t sort_tmp, o_kin, o_kout, o_vin, total;
};

cudaError_t order_plan(int64_t n, int64_t n_base, OrderPlan& p) {
  const int64_t max_key = (n_base > 0 ? n_base : 1) * 256;
  p.end_bit = end_bit_for(max_key);
  p.narrow = p.end_bit <= 32;
  const size_t kb = p.narrow ? 4 : 8;
  p.sort_tmp = 0;
  cudaError_t e = p.narrow
      ? cub::DeviceRadixSort::SortPairs(nullptr, p.sort_tmp, (const uint32_t*)nullptr,
                                        (uint32_t*)nullptr, (const int32_t*)nullptr,
                                        (int32_t*)nullptr, (int)n, 0, p.end_bit)
      : cub::DeviceRadixSort::SortPairs(nullptr, p.sort_tmp, (const uint64_t*)nullptr,
                                        (uint64_t*)nullptr, (const int32_t*)nullptr,
                                        (int32_t*)nullptr, (int)n, 0, p.end_bit);
  p.o_kin = 0;
  p.o_kout = align256(p.o_kin + kb * n);
  p.o_vin = align256(p.o_kout + kb * n);
  p.total = align256(p.o_vin + 4 * n) + p.sort_tmp;
  return e;
}

struct IndexPlan {
  int64_t rows, nt, nn, wide_total;
  int wide_levels;
  int64_t wide_off[8], wide_cnt[8];
  int depth_max;
  // arena offsets
  size_t a_rec, a_rec32, a_pairs, a_perm, a_inv, a_tbox, a_tbox32, a_nbox, a_nbox32, a_ncb32,
      a_range, a_wide32, a_recB, a_recU, a_stats, arena;
  // workspace offsets
  size_t w_key, w_key2, w_val, w_val2, w_seg, w_seg2, w_id, w_order, w_bbox, w_wide, w_lvl,
      w_tmp, sort_tmp, workspace;
};

int index_plan(int64_t n, int d, int flags, IndexPlan& P) {
  if (n < 1 || n >= ((int64_t)1 << 31) - VR_REC_PAD || d < VR_MIN_D || d > VR_MAX_D)
    return d < VR_MIN_D || d > VR_MAX_D ? VR_EDIM : VR_EINVAL;
  P.rows = rec_rows(n);
  P.nt = (n + TILE - 1) / TILE;
  int64_t size = 1;
  while (size < P.nt) size *= 2;
  P.nn = 2 * size - 1;
  P.depth_max = 0;
  while (((int64_t)1 << P.depth_max) < P.nt) ++P.depth_max;  // ceil(log2 nt)
  // 32-ary levels: tiles, then unions of 32, ..., one root (at least two)
  int64_t m = P.nt;
  P.wide_levels = 0;
  int64_t off = 0;
  while (true) {
    if (P.wide_levels >= 8) return VR_EINVAL;
    P.wide_off[P.wide_levels] = off;
    P.wide_cnt[P.wide_levels] = m;
    off += m;
    ++P.wide_levels;
    if (m == 1 && P.wide_levels >= 2) break;
    m = (m + WIDE - 1) / WIDE;
  }
  for (int l = P.wide_levels; l < 8; ++l) P.wide_off[l] = P.wide_cnt[l] = 0;
  P.wide_total = off;
  const int S = rec_stride(d), S32 = rec32_stride(d), P2 = rec32p_stride(d),
            B32 = box32_stride(d), KS = (d + 2 + 7) / 8;
  size_t a = 0;
  P.a_rec = a;     a = align256(a + sizeof(double) * P.rows * S);
  P.a_rec32 = a;   a = align256(a + sizeof(float) * P.rows * S32);
  P.a_pairs = a;   a = align256(a + sizeof(float) * (P.rows / 2) * P2);
  P.a_perm = a;    a = align256(a + sizeof(int32_t) * n);
  P.a_inv = a;     a = align256(a + sizeof(int32_t) * n);
  P.a_tbox = a;    a = align256(a + sizeof(double) * P.nt * 2 * d);
  P.a_tbox32 = a;  a = align256(a + sizeof(float) * P.nt * B32);
  P.a_nbox = a;    a = align256(a + sizeof(double) * P.nn * 2 * d);
  P.a_nbox32 = a;  a = align256(a + sizeof(float) * P.nn * B32);
  P.a_ncb32 = a;   a = align256(a + sizeof(float) * P.nn * B32);
  P.a_range = a;   a = align256(a + sizeof(int32_t) * P.nn * 2);
  P.a_wide32 = a;  a = align256(a + sizeof(float) * P.wide_total * B32);
  P.a_recB = a;
  if (flags & VR_PRUNE_MMA) a = align256(a + sizeof(float) * P.rows * 8 * KS);
  P.a_recU = a;
  if (flags & VR_PRUNE_UMMA) a = align256(a + sizeof(float) * P.rows * 8 * KS);
  P.a_stats = a;   a = align256(a + sizeof(double) * 32);
  P.arena = a;
  // build scratch
  P.sort_tmp = 0;
  size_t t1 = 0, t2 = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(
      nullptr, t1, (const double*)nullptr, (double*)nullptr, (const unsigned long long*)nullptr,
      (unsigned long long*)nullptr, (int)n);
  if (e != cudaSuccess) return vr_cuda_status(e);
  e = cub::DeviceRadixSort::SortPairs(nullptr, t2, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                      (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  if (e != cudaSuccess) return vr_cuda_status(e);
  P.sort_tmp = t1 > t2 ? t1 : t2;
  const int64_t level_nodes = P.depth_max > 0 ? ((int64_t)1 << (P.depth_max - 1)) : 1;
  size_t w = 0;
  P.w_key = w;    w = align256(w + sizeof(double) * n);
  P.w_key2 = w;   w = align256(w + sizeof(double) * n);
  P.w_val = w;    w = align256(w + sizeof(uint64_t) * n);
  P.w_val2 = w;   w = align256(w + sizeof(uint64_t) * n);
  P.w_seg = w;    w = align256(w + sizeof(uint32_t) * n);
  P.w_seg2 = w;   w = align256(w + sizeof(uint32_t) * n);
  P.w_id = w;     w = align256(w + sizeof(int32_t) * n);
  P.w_order = w;  w = align256(w + sizeof(int32_t) * n);
  P.w_bbox = w;   w = align256(w + sizeof(uint64_t) * level_nodes * 2 * d);
  P.w_wide = w;   w = align256(w + sizeof(double) * P.wide_total * 2 * d);
  P.w_lvl = w;    w = align256(w + sizeof(int64_t) * 16);
  P.w_tmp = w;    w = align256(w + P.sort_tmp);
  P.workspace = w;
  return VR_OK;
}

}  // namespace

extern "C" int vr_screen32_stats(const double* rec, int64_t n, int d, const double* center,
                                 double* stats, void* stream) {
  if (!rec || !stats || n < 1) return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  unsigned long long* mm = reinterpret_cast<unsigned long long*>(stats + 16);
  const unsigned nb = grid_for(n, 256, 1184);
  VR_DISPATCH_D(d, {
    if (!center) {
      k_fill_u64<<<1, 32, 0, st>>>(mm, 16, 0xffffffffffffffffull, 0ull);
      k_stats_minmax<D><<<nb, 256, 0, st>>>(rec, n, mm);
    }
    k_stats_centre<D><<<1, 32, 0, st>>>(stats, center);
    k_stats_spread<D><<<nb, 256, 0, st>>>(rec, n, stats);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_prune_index_layout(int64_t n, int d, int flags, vr_prune_layout* out) {
  if (!out) return VR_EINVAL;
  IndexPlan P;
  const int s = index_plan(n, d, flags, P);
  if (s) return s;
  out->arena_bytes = (int64_t)P.arena;
  out->workspace_bytes = (int64_t)P.workspace;
  out->n_tiles = P.nt;
  out->n_nodes = P.nn;
  out->wide_levels = P.wide_levels;
  return VR_OK;
}

extern "C" int vr_build_prune_index(const double* rec, int64_t n, int d, const double* center,
                                    int flags, void* arena, int64_t arena_bytes, void* workspace,
                                    int64_t workspace_bytes, vr_prune_index* out, void* stream) {
  if (!rec || !center || !arena || !workspace || !out) return VR_EINVAL;
  IndexPlan P;
  int s = index_plan(n, d, flags, P);
  if (s) return s;
  if (arena_bytes < (int64_t)P.arena || workspace_bytes < (int64_t)P.workspace)
    return VR_ECAPACITY;
  cudaStream_t st = as_stream(stream);
  char* A = static_cast<char*>(arena);
  char* W = static_cast<char*>(workspace);
  double* crec = reinterpret_cast<double*>(A + P.a_rec);
  float* rec32 = reinterpret_cast<float*>(A + P.a_rec32);
  float* pairs = reinterpret_cast<float*>(A + P.a_pairs);
  int32_t* perm = reinterpret_cast<int32_t*>(A + P.a_perm);
  int32_t* inv = reinterpret_cast<int32_t*>(A + P.a_inv);
  double* tbox = reinterpret_cast<double*>(A + P.a_tbox);
  float* tbox32 = reinterpret_cast<float*>(A + P.a_tbox32);
  double* nbox = reinterpret_cast<double*>(A + P.a_nbox);
  float* nbox32 = reinterpret_cast<float*>(A + P.a_nbox32);
  float* ncb32 = reinterpret_cast<float*>(A + P.a_ncb32);
  int32_t* range = reinterpret_cast<int32_t*>(A + P.a_range);
  float* wide32 = reinterpret_cast<float*>(A + P.a_wide32);
  float* recB = (flags & VR_PRUNE_MMA) ? reinterpret_cast<float*>(A + P.a_recB) : nullptr;
  float* recU = (flags & VR_PRUNE_UMMA) ? reinterpret_cast<float*>(A + P.a_recU) : nullptr;
  double* cdev = reinterpret_cast<double*>(A + P.a_stats);
  double* key = reinterpret_cast<double*>(W + P.w_key);
  double* key2 = reinterpret_cast<double*>(W + P.w_key2);
  unsigned long long* val = reinterpret_cast<unsigned long long*>(W + P.w_val);
  unsigned long long* val2 = reinterpret_cast<unsigned long long*>(W + P.w_val2);
  uint32_t* seg = reinterpret_cast<uint32_t*>(W + P.w_seg);
  uint32_t* seg2 = reinterpret_cast<uint32_t*>(W + P.w_seg2);
  int32_t* ids = reinterpret_cast<int32_t*>(W + P.w_id);
  int32_t* order = reinterpret_cast<int32_t*>(W + P.w_order);
  unsigned long long* bbox = reinterpret_cast<unsigned long long*>(W + P.w_bbox);
  double* widescr = reinterpret_cast<double*>(W + P.w_wide);
  int64_t* lvl = reinterpret_cast<int64_t*>(W + P.w_lvl);
  void* tmp = W + P.w_tmp;
  cudaError_t e;
  // the centre is copied into the arena (the caller's buffer may be transient)
  if ((e = cudaMemcpyAsync(cdev, center, sizeof(double) * d, cudaMemcpyDeviceToDevice, st)) !=
      cudaSuccess)
    return vr_cuda_status(e);
  int64_t lvl_host[16];
  for (int l = 0; l < 8; ++l) { lvl_host[l] = P.wide_off[l]; lvl_host[8 + l] = P.wide_cnt[l]; }
  // pageable source: the copy is staged before cudaMemcpyAsync returns
  if ((e = cudaMemcpyAsync(lvl, lvl_host, sizeof(lvl_host), cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return vr_cuda_status(e);
  k_node_ranges<<<grid_for(P.nn), 256, 0, st>>>(P.nn, P.nt, range);
  k_iota32<<<grid_for(n), 256, 0, st>>>(order, n);
  const int seg_bits = end_bit_for(P.nt);
  VR_DISPATCH_D(d, {
    for (int depth = 0; depth < P.depth_max; ++depth) {
      const int64_t nodes = (int64_t)1 << depth;
      k_fill_u64<<<grid_for(nodes * 2 * D), 256, 0, st>>>(bbox, nodes * 2 * D,
                                                          0xffffffffffffffffull, 0ull);
      k_level_bbox<D><<<grid_for(n, 256, 4096), 256, 0, st>>>(rec, order, n, P.nt, depth, bbox);
      k_level_keys<D><<<grid_for(n, 256, 4096), 256, 0, st>>>(rec, order, n, P.nt, depth, bbox,
                                                              key, val);
      size_t t = P.sort_tmp;
      e = cub::DeviceRadixSort::SortPairs(tmp, t, key, key2, val, val2, (int)n, 0, 64, st);
      if (e != cudaSuccess) return vr_cuda_status(e);
      k_split_val<<<grid_for(n, 256, 4096), 256, 0, st>>>(val2, n, seg, ids);
      t = P.sort_tmp;
      e = cub::DeviceRadixSort::SortPairs(tmp, t, seg, seg2, ids, order, (int)n, 0, seg_bits, st);
      if (e != cudaSuccess) return vr_cuda_status(e);
    }
    k_gather<D><<<grid_for(P.rows, 256, 4096), 256, 0, st>>>(rec, order, n, P.rows, crec, perm,
                                                             inv);
    k_tile_box<D><<<grid_for(P.nt * 32, 256, 4096), 256, 0, st>>>(crec, n, P.nt, tbox);
    k_tile_box32<D><<<grid_for(P.nt), 256, 0, st>>>(tbox, P.nt, cdev, tbox32);
    k_node_box<D><<<grid_for(P.nn * 32, 256, 4096), 256, 0, st>>>(tbox, range, P.nn, cdev, nbox,
                                                                   nbox32, ncb32);
    k_wide_box32<D><<<grid_for(P.wide_total * 32, 256, 4096), 256, 0, st>>>(
        tbox, P.nt, P.wide_levels, lvl, cdev, wide32, widescr);
  });
  if ((e = cudaGetLastError()) != cudaSuccess) return vr_cuda_status(e);
  if ((s = vr_pack_records32(crec, P.rows, d, cdev, rec32, stream))) return s;
  if ((s = vr_pack_records32_pairs(rec32, P.rows, d, pairs, stream))) return s;
  if (recB && (s = vr_pack_records_mma(rec32, P.rows, d, recB, stream))) return s;
  if (recU && (s = vr_pack_records_umma(rec32, P.rows, d, recU, stream))) return s;
  out->rec = crec;
  out->rec32 = pairs;
  out->perm = perm;
  out->inv_perm = inv;
  out->tile_box = tbox;
  out->tile_box32 = tbox32;
  out->node_box = nbox;
  out->node_box32 = nbox32;
  out->node_range = range;
  out->n = n;
  out->wide_box32 = wide32;
  out->wide_levels = P.wide_levels;
  for (int l = 0; l < 8; ++l) {
    out->wide_off[l] = P.wide_off[l];
    out->wide_cnt[l] = P.wide_cnt[l];
  }
  out->recB = recB;
  out->rec32rows = rec32;
  out->node_cb32 = ncb32;
  out->recU = recU;
  return VR_OK;
}

extern "C" int vr_ray_keys(const int32_t* inv_perm, const int32_t* eta, int eta_len,
                           int64_t rays_per_cell, const double* u, int64_t n, int d,
                           int64_t* keys, void* stream) {
  if (n <= 0) return VR_OK;
  if (!u || !keys || (eta && (!inv_perm || eta_len < 1)) || (!eta && rays_per_cell < 1))
    return VR_EINVAL;
  VR_DISPATCH_D(d, {
    k_ray_keys<D, int64_t><<<grid_for(n), 256, 0, as_stream(stream)>>>(
        inv_perm, eta, eta_len, rays_per_cell, u, n, keys, nullptr);
  });
  VR_RETURN_LAUNCH();
}

extern "C" int vr_ray_order(const int32_t* inv_perm, const int32_t* eta, int eta_len,
                            int64_t rays_per_cell, const double* u, int64_t n, int d,
                            int64_t n_base, int32_t* order, void* workspace,
                            int64_t* workspace_bytes, void* stream) {
  if (!workspace_bytes || n < 0 || n >= ((int64_t)1 << 31)) return VR_EINVAL;
  OrderPlan p;
  cudaError_t e = order_plan(n > 0 ? n : 1, n_base, p);
  if (e != cudaSuccess) return vr_cuda_status(e);
  if (!workspace) {
    *workspace_bytes = (int64_t)p.total;
    return VR_OK;
  }
  if (*workspace_bytes < (int64_t)p.total) return VR_ECAPACITY;
  if (n == 0) return VR_OK;
  if (!u || !order || (eta && (!inv_perm || eta_len < 1)) || (!eta && rays_per_cell < 1))
    return VR_EINVAL;
  cudaStream_t st = as_stream(stream);
  char* W = static_cast<char*>(workspace);
  int32_t* vin = reinterpret_cast<int32_t*>(W + p.o_vin);
  void* tmp = W + align256(p.o_vin + 4 * n);
  size_t t = p.sort_tmp;
  VR_DISPATCH_D(d, {
    if (p.narrow) {
      uint32_t* kin = reinterpret_cast<uint32_t*>(W + p.o_kin);
      uint32_t* kout = reinterpret_cast<uint32_t*>(W + p.o_kout);
      k_ray_keys<D, uint32_t><<<grid_for(n), 256, 0, st>>>(inv_perm, eta, eta_len, rays_per_cell,
                                                            u, n, kin, vin);
      e = cub::DeviceRadixSort::SortPairs(tmp, t, kin, kout, vin, order, (int)n, 0, p.end_bit, st);
    } else {
      uint64_t* kin = reinterpret_cast<uint64_t*>(W + p.o_kin);
      uint64_t* kout = reinterpret_cast<uint64_t*>(W + p.o_kout);
      k_ray_keys<D, uint64_t><<<grid_for(n), 256, 0, st>>>(inv_perm, eta, eta_len, rays_per_cell,
                                                            u, n, kin, vin);
      e = cub::DeviceRadixSort::SortPairs(tmp, t, kin, kout, vin, order, (int)n, 0, p.end_bit, st);
    }
  });
  if (e != cudaSuccess) return vr_cuda_status(e);
  VR_RETURN_LAUNCH();
}
