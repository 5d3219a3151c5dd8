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
#include "trav_core.cuh"

namespace {

inline unsigned nb(int64_t n, int nt = 256) { return (unsigned)((n + nt - 1) / nt); }

Tables from(const vr_traverse_tables* p) {
  return Tables{p->vkeys, p->vstate, p->vval, p->vlevel, p->vcap,
                p->ekeys, p->estate, p->ecount, p->ecap, p->overflow};
}

bool pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

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

extern "C" int vr_trav_open_edges(const vr_traverse_tables* tab, int d, const int32_t* sigma,
                                  int64_t n_v, uint8_t* open_mask, int32_t* open_count,
                                  void* stream) {
  if (!tab || !sigma || !open_mask || !open_count) return VR_EINVAL;
  if (n_v <= 0) return VR_OK;
  const Tables t = from(tab);
  VR_DISPATCH_D_ALL(d, {
    k_open_edges<D><<<nb(n_v, 128), 128, 0, as_stream(stream)>>>(t, sigma, n_v, open_mask,
                                                                  open_count);
  });
  VR_RETURN_LAUNCH();
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
