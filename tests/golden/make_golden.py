"""Generate the golden fixtures by running the UNMODIFIED reference.

Build-container only: imports the read-only reference from
/root/reference/pkg/src.  The .npz outputs are committed next to this
script; nothing on the GPU box reads /root/reference.

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Fixtures (inputs are regenerated from their numpy seeds, which are stable):
  config2_sample.npz  first K canonical config-2 rays: the
                      descent vertices they start from and the reference
                      raycast_incircle results.
  config5_sample.npz  N=1e6, d=8 fp32-upcast: generator-start rays and the
                      edge rays of 10 descent vertices (kd-tree path).
  mesh_config1.npz    voronoi_graph on config 1 (N=1000, d=3, seed 0).
  meshes_small.npz    the reference test-suite instances (conftest.py,
                      test_graph.py, test_raycast.py).
  mc_golden.npz       mc_areas_only under replayed normals (config-4 cells,
                      unit square, neighbour-restricted path).
"""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

import voronray as vr  # noqa: E402
from voronray import rng as vrng  # noqa: E402
from voronray.errors import DegenerateConfiguration, UnboundedRay  # noqa: E402
from voronray.raycast import _vertex_directions  # noqa: E402

from oracle.voronray_oracle import philox_normals  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


class Replay:
    def __init__(self, z):
        self.z = np.asarray(z, dtype=float).ravel()
        self.pos = 0

    def standard_normal(self, size=None):
        m = 1 if size is None else int(np.prod(size))
        out = self.z[self.pos:self.pos + m]
        self.pos += m
        return float(out[0]) if size is None else out.reshape(size).copy()


def cast(ns, eta, x, u):
    """(status, idx, rp): status 0 ok, 1 escaped, 3 degenerate."""
    try:
        res = vr.raycast_incircle(ns, vr.RayQuery(tuple(int(e) for e in eta), x, u), heuristic=False)
    except DegenerateConfiguration:
        return 3, -1, np.full(ns.dim, np.nan)
    if res is None:
        return 1, -1, np.full(ns.dim, np.nan)
    sig, rp = res
    new = [s for s in sig if s not in set(int(e) for e in eta)]
    return 0, int(new[0]), np.asarray(rp)


def config2_rays(k):
    """Canonical config-2 ray recipe, first k rays."""
    s = np.random.default_rng(1).choice(20000, 10000, replace=False)
    p = np.random.default_rng(2).integers(0, 10000, 10 ** 6)[:k]
    u = np.random.default_rng(3).standard_normal((10 ** 6, 6))[:k]
    u = u / np.linalg.norm(u, axis=1, keepdims=True)
    return s, p, u


def config2_sample(k=4000):
    pts = np.random.default_rng(0).random((20000, 6))
    ns = vr.build_node_set(pts)
    s, p, u = config2_rays(k)
    need = np.unique(p)
    t0 = time.time()
    vsig = np.zeros((len(need), 7), dtype=np.int32)
    vr_ = np.zeros((len(need), 6))
    for m, pp in enumerate(need):
        v = vr.descent(ns, int(s[pp]), vrng.stream(0, "descent", int(s[pp])))
        vsig[m] = v.sigma
        vr_[m] = v.r
    t_desc = time.time() - t0
    pos = {int(pp): m for m, pp in enumerate(need)}
    x = np.array([vr_[pos[int(pp)]] for pp in p])
    sig_k = np.array([vsig[pos[int(pp)]] for pp in p])
    proj = np.einsum("kd,ksd->ks", u, pts[sig_k])
    g = sig_k[np.arange(k), np.argmax(proj, axis=1)]
    t0 = time.time()
    status = np.zeros(k, dtype=np.int8)
    idx = np.zeros(k, dtype=np.int64)
    rp = np.zeros((k, 6))
    for m in range(k):
        status[m], idx[m], rp[m] = cast(ns, (g[m],), x[m], u[m])
    t_ray = time.time() - t0
    np.savez_compressed(os.path.join(HERE, "config2_sample.npz"), pool_p=need,
                        pool_start=s[need], pool_sigma=vsig, pool_r=vr_, ray_p=p, u=u, g=g,
                        status=status, idx=idx, rp=rp)
    print("config2", k, "rays; escapes", int((status == 1).sum()), "degenerate",
          int((status == 3).sum()), f"descent {t_desc:.1f}s rays {t_ray:.1f}s "
          f"({k / t_ray:.0f} rays/s)")


def config5_sample(n_gen_rays=200, n_seeds=10):
    pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    t0 = time.time()
    ns = vr.build_node_set(pts)
    print("config5 nodeset", time.time() - t0)
    rg = np.random.default_rng(4)
    g = rg.choice(10 ** 6, n_gen_rays, replace=False)
    u = np.random.default_rng(5).standard_normal((n_gen_rays, 8))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    gs = np.zeros(n_gen_rays, dtype=np.int8)
    gi = np.zeros(n_gen_rays, dtype=np.int64)
    grp = np.zeros((n_gen_rays, 8))
    t0 = time.time()
    for m in range(n_gen_rays):
        gs[m], gi[m], grp[m] = cast(ns, (g[m],), pts[g[m]], u[m])
    print("config5 gen rays", time.time() - t0)
    seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)[:n_seeds]
    vsig = np.zeros((n_seeds, 9), dtype=np.int32)
    vrr = np.zeros((n_seeds, 8))
    e_x, e_u, e_eta, e_st, e_i, e_rp = [], [], [], [], [], []
    t0 = time.time()
    for m, sd in enumerate(seeds):
        v = vr.descent(ns, int(sd), vrng.stream(0, "descent", int(sd)))
        vsig[m], vrr[m] = v.sigma, v.r
        dirs = _vertex_directions(ns.points, v.sigma, range(9))
        for kk in range(9):
            eta = v.sigma[:kk] + v.sigma[kk + 1:]
            st, i, rp = cast(ns, eta, v.r, dirs[kk])
            e_x.append(v.r)
            e_u.append(dirs[kk])
            e_eta.append(eta)
            e_st.append(st)
            e_i.append(i)
            e_rp.append(rp)
    print("config5 descents+edges", time.time() - t0)
    np.savez_compressed(os.path.join(HERE, "config5_sample.npz"), gen_g=g, gen_u=u, gen_status=gs,
                        gen_idx=gi, gen_rp=grp, seeds=seeds, seed_sigma=vsig, seed_r=vrr,
                        edge_x=np.array(e_x), edge_u=np.array(e_u),
                        edge_eta=np.array(e_eta, dtype=np.int32),
                        edge_status=np.array(e_st, dtype=np.int8), edge_idx=np.array(e_i),
                        edge_rp=np.array(e_rp))


def mesh_arrays(mesh):
    keys = sorted(mesh.vertices)
    sig = np.array(keys, dtype=np.int32)
    r = np.array([mesh.vertices[k].r for k in keys])
    bnd = sorted((b.sigma, tuple(b.u)) for b in mesh.boundary)
    bs = np.array([b[0] for b in bnd], dtype=np.int32).reshape(len(bnd), -1)
    bu = np.array([b[1] for b in bnd]).reshape(len(bnd), -1)
    ek = sorted(mesh.edge_counts)
    ekeys = np.array(ek, dtype=np.int32)
    ecnt = np.array([mesh.edge_counts[e] for e in ek], dtype=np.int32)
    return sig, r, bs, bu, ekeys, ecnt


def mesh_config1():
    pts = np.random.default_rng(0).random((1000, 3))
    stats = vr.RaycastStats()
    t0 = time.time()
    mesh = vr.voronoi_graph(vr.build_node_set(pts), seed=0, stats=stats)
    wall = time.time() - t0
    sig, r, bs, bu, ek, ec = mesh_arrays(mesh)
    np.savez_compressed(os.path.join(HERE, "mesh_config1.npz"), sigma=sig, r=r, boundary_sigma=bs,
                        boundary_u=bu, edge_key=ek, edge_count=ec, raycasts=stats.raycasts,
                        nn_calls=stats.nn_calls, wall_s=wall)
    dig = hashlib.sha256(np.ascontiguousarray(sig, dtype="<i4").tobytes()).hexdigest()
    print("config1 V", len(sig), "B", len(bs), "digest", dig, f"{wall:.2f}s")


SMALL = {
    # name: (points recipe, voronoi_graph seed)
    "mesh_2d": (lambda: np.random.default_rng(1234).random((120, 2)), 0),
    "mesh_3d": (lambda: np.random.default_rng(999).random((90, 3)), 0),
    "four_point": (lambda: np.array([(0.0, 0.0), (2.0, 0.0), (0.0, 2.0), (2.0, 2.1)]), 42),
    "unit_square": (lambda: np.array([(0.0, 0.0), (1.0, 0.0), (-1.0, 0.0), (0.0, 1.0),
                                      (0.0, -1.0)]), 3),
    "nodup_d2": (lambda: np.random.default_rng(25).random((300, 2)), 0),
    "nodup_d3": (lambda: np.random.default_rng(26).random((300, 3)), 0),
    "incircle_d4": (lambda: np.random.default_rng(14).random((1000, 4)), 0),
    "incircle_d5": (lambda: np.random.default_rng(15).random((500, 5)), 0),
    "oracle_3d_50": (lambda: np.random.default_rng(17).random((50, 3)), 5),
    "gauss_d5_2000": (lambda: np.random.default_rng(0).standard_normal((2000, 5)), 0),
}


def meshes_small():
    out = {}
    for name, (mk, seed) in SMALL.items():
        pts = mk()
        stats = vr.RaycastStats()
        mesh = vr.voronoi_graph(vr.build_node_set(pts), seed=seed, stats=stats)
        sig, r, bs, bu, ek, ec = mesh_arrays(mesh)
        out[f"{name}__sigma"] = sig
        out[f"{name}__r"] = r
        out[f"{name}__boundary_sigma"] = bs
        out[f"{name}__edge_key"] = ek
        out[f"{name}__edge_count"] = ec
        out[f"{name}__raycasts"] = np.array(stats.raycasts)
        print(name, len(sig), "vertices", len(bs), "boundary")
    np.savez_compressed(os.path.join(HERE, "meshes_small.npz"), **out)


def mc_golden():
    out = {}
    # (a) config-4 cells under the device Philox stream (numpy port)
    pts = np.random.default_rng(0).random((100000, 4))
    ns = vr.build_node_set(pts)
    order = np.argsort(np.linalg.norm(pts - 0.5, axis=1), kind="stable")
    cells = order[:8]
    z = philox_normals(0, cells, 1000, 4)
    vols, fj, fa, fo = [], [], [], [0]
    t0 = time.time()
    for m, c in enumerate(cells):
        areas, vol = vr.mc_areas_only(ns, int(c), 1000, Replay(z[m * 1000:(m + 1) * 1000]))
        vols.append(vol)
        for j in sorted(areas):
            fj.append(j)
            fa.append(areas[j])
        fo.append(len(fj))
    print("mc config4 cells", time.time() - t0)
    out.update(c4_cells=cells, c4_z=z, c4_volume=np.array(vols), c4_face_j=np.array(fj),
               c4_face_area=np.array(fa), c4_face_off=np.array(fo))
    # (b) unit square, reference test stream (test_integrate_mc.py:63-67)
    usq = vr.build_node_set([(0.0, 0.0), (1.0, 0.0), (-1.0, 0.0), (0.0, 1.0), (0.0, -1.0)])
    areas, vol, smp = vr.mc_areas_only(usq, 0, 20000, vrng.stream(2024, "test", 4),
                                       return_samples=True)
    out.update(usq_face_j=np.array(sorted(areas)), usq_face_area=np.array([areas[j] for j in sorted(areas)]),
               usq_volume=np.array(vol), usq_samples=smp)
    # (c) mesh_2d bounded cell, neighbour-restricted batch path
    m2 = vr.voronoi_graph(vr.build_node_set(np.random.default_rng(1234).random((120, 2))), seed=0)
    i = m2.bounded_cells()[2]
    nb = np.asarray(m2.neighbors(i), dtype=np.intp)
    areas, vol = vr.mc_areas_only(m2.nodes, i, 3000, vrng.stream(2024, "test", 20), neighbors=nb)
    out.update(m2_cell=np.array(i), m2_neighbors=nb, m2_face_j=np.array(sorted(areas)),
               m2_face_area=np.array([areas[j] for j in sorted(areas)]), m2_volume=np.array(vol))
    # (d) unbounded cell: first escaping direction (test_integrate_mc.py:99-103)
    try:
        vr.mc_areas_only(usq, 1, 2000, vrng.stream(2024, "test", 8))
    except UnboundedRay as e:
        out.update(unb_cell=np.array(e.cell), unb_dir=np.asarray(e.direction))
    np.savez_compressed(os.path.join(HERE, "mc_golden.npz"), **out)


def config5_balls(n_seeds=5, hops=4):
    """Reference-computed L-hop vertex balls around descent vertices at
    N=1e6, d=8 (fp32-upcast uniform): BFS over the vertex-edge graph, every
    edge raycast with the unmodified reference raycast_incircle."""
    pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    ns = vr.build_node_set(pts)
    seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)[:n_seeds]
    out = {}
    t0 = time.time()
    for m, sd in enumerate(seeds):
        v = vr.descent(ns, int(sd), vrng.stream(0, "descent", int(sd)))
        dist = {v.sigma: 0}
        coords = {v.sigma: v.r}
        frontier = [v.sigma]
        for h in range(1, hops + 1):
            nxt = []
            for sig in frontier:
                dirs = _vertex_directions(ns.points, sig, range(9))
                for k in range(9):
                    eta = sig[:k] + sig[k + 1:]
                    res = vr.raycast_incircle(ns, vr.RayQuery(eta, coords[sig], dirs[k]),
                                              heuristic=False)
                    if res is None:
                        continue
                    s2, r2 = res
                    if s2 not in dist:
                        dist[s2] = h
                        coords[s2] = r2
                        nxt.append(s2)
            frontier = nxt
        keys = sorted(dist)
        out[f"seed{m}"] = np.array([int(sd)])
        out[f"ball{m}_sigma"] = np.array(keys, dtype=np.int32)
        out[f"ball{m}_hops"] = np.array([dist[k] for k in keys], dtype=np.int8)
        print("config5 ball", m, len(keys), "vertices", f"{time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "config5_balls.npz"), **out)


_C5_NS = None


def _c5_ball(args):
    """One seed's L-hop ball (BFS, every edge raycast by the reference)."""
    m, sd, hops = args
    ns = _C5_NS
    t0 = time.time()
    v = vr.descent(ns, int(sd), vrng.stream(0, "descent", int(sd)))
    dist = {v.sigma: 0}
    coords = {v.sigma: v.r}
    frontier = [v.sigma]
    for h in range(1, hops + 1):
        nxt = []
        for sig in frontier:
            dirs = _vertex_directions(ns.points, sig, range(9))
            for k in range(9):
                eta = sig[:k] + sig[k + 1:]
                res = vr.raycast_incircle(ns, vr.RayQuery(eta, coords[sig], dirs[k]),
                                          heuristic=False)
                if res is None:
                    continue
                s2, r2 = res
                if s2 not in dist:
                    dist[s2] = h
                    coords[s2] = r2
                    nxt.append(s2)
        frontier = nxt
    keys = sorted(dist)
    print("config5 L5 ball", m, len(keys), "vertices", f"{time.time() - t0:.1f}s", flush=True)
    return (m, int(sd), np.array(keys, dtype=np.int32),
            np.array([dist[k] for k in keys], dtype=np.int8),
            np.array([coords[k] for k in keys]))


def config5_balls_l5(n_seeds=20, hops=5, procs=8):
    """SURVEY.md §8(d) config-5 pin at bench scale: the L=5 balls of the
    first 20 canonical seeds (reference descent + raycast_incircle BFS, as
    config5_balls above), one process per seed with the NodeSet fork-shared.
    The GPU test asserts every ball is contained in the 10,000-seed L=5
    vertex set (and equals the GPU's own ball of that seed)."""
    import multiprocessing as mp
    global _C5_NS
    pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    _C5_NS = vr.build_node_set(pts)
    seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)[:n_seeds]
    t0 = time.time()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_c5_ball, [(m, int(sd), hops) for m, sd in enumerate(seeds)], chunksize=1)
    out = {"hops": np.array([hops]), "seeds": seeds.astype(np.int64)}
    for m, sd, sig, hp, r in res:
        out[f"ball{m}_sigma"] = sig
        out[f"ball{m}_hops"] = hp
        out[f"ball{m}_r"] = r
    out["reference_wall_s"] = np.array([time.time() - t0])
    out["procs"] = np.array([procs])
    np.savez_compressed(os.path.join(HERE, "config5_balls_l5.npz"), **out)


def mc_integrate_golden():
    """mc_integrate_cell with the reference's built-in integrands and a plain
    Python callable, on reference RNG streams (integrate_mc.py:70-121)."""
    from voronray.integrands import const1, sinx2, make_linear
    out = {}
    usq = vr.build_node_set([(0.0, 0.0), (1.0, 0.0), (-1.0, 0.0), (0.0, 1.0), (0.0, -1.0)])
    cases = []
    res = vr.mc_integrate_cell(usq, 0, const1, 20000, 2, vrng.stream(2024, "test", 3))
    cases.append(("usq_const1", res))
    res = vr.mc_integrate_cell(usq, 0, make_linear([1.0, -2.0, 0.5]), 5000, 3,
                               vrng.stream(2024, "test", 6))
    cases.append(("usq_linear", res))
    m2 = vr.voronoi_graph(vr.build_node_set(np.random.default_rng(1234).random((120, 2))), seed=0)
    i = m2.bounded_cells()[2]
    nb = np.asarray(m2.neighbors(i), dtype=np.intp)
    res = vr.mc_integrate_cell(m2.nodes, i, lambda x: x[0], 2000, 2, vrng.stream(2024, "test", 20))
    cases.append(("m2_x0_full", res))
    res = vr.mc_integrate_cell(m2.nodes, i, lambda x: x[0], 2000, 2, vrng.stream(2024, "test", 20),
                               neighbors=nb)
    cases.append(("m2_x0_nb", res))
    pts = np.random.default_rng(0).random((100000, 4))
    ns = vr.build_node_set(pts)
    order = np.argsort(np.linalg.norm(pts - 0.5, axis=1), kind="stable")
    for c in order[:2]:
        res = vr.mc_integrate_cell(ns, int(c), sinx2, 1000, 3, vrng.stream(7, "mc", int(c)))
        cases.append((f"c4_sinx2_{int(c)}", res))
    out["m2_cell"] = np.array(i)
    for name, r in cases:
        js = sorted(r.area)
        out[f"{name}__j"] = np.array(js)
        out[f"{name}__area"] = np.array([r.area[j] for j in js])
        out[f"{name}__surf"] = np.array([r.surface_integral[j] for j in js])
        out[f"{name}__vol"] = np.array([r.volume, r.volume_integral])
        print(name, r.volume, r.volume_integral, len(js))
    np.savez_compressed(os.path.join(HERE, "mc_integrate_golden.npz"), **out)


def hmc_io_golden():
    """HMC post-processing and the mesh JSON wire format on mesh_2d
    (integrate_hmc.py, io.py), with reference MC areas."""
    from voronray.integrands import sinx2
    from voronray.integrate_hmc import hmc_cell_integral, hmc_interface_integral, hmc_volume
    from voronray.io import mesh_to_dict
    import json
    m2 = vr.voronoi_graph(vr.build_node_set(np.random.default_rng(1234).random((120, 2))), seed=0)
    out = {}
    cells = m2.bounded_cells()[:6]
    for c in cells:
        nb = np.asarray(m2.neighbors(c), dtype=np.intp)
        areas, vol = vr.mc_areas_only(m2.nodes, c, 4000, vrng.stream(5, "mc", c), neighbors=nb)
        js = sorted(areas)
        out[f"c{c}__j"] = np.array(js)
        out[f"c{c}__area"] = np.array([areas[j] for j in js])
        hv = hmc_volume(m2.nodes, c, areas, m2)
        fi = [hmc_interface_integral(m2, c, j, areas[j], sinx2) for j in js]
        ci = hmc_cell_integral(m2, c, sinx2, areas, hv)
        out[f"c{c}__hmc"] = np.array([hv, ci])
        out[f"c{c}__face"] = np.array(fi)
    out["cells"] = np.array(cells)
    d = mesh_to_dict(m2)
    out["mesh_json_sha"] = np.frombuffer(
        hashlib.sha256(json.dumps(d, indent=1, sort_keys=True).encode()).digest(), dtype=np.uint8)
    out["n_json_vertices"] = np.array(len(d["vertices"]))
    np.savez_compressed(os.path.join(HERE, "hmc_io_golden.npz"), **out)
    print("hmc/io cells", cells)


if __name__ == "__main__":
    which = sys.argv[1:] or ["mesh_config1", "meshes_small", "config2_sample", "mc_golden",
                             "config5_sample"]
    for w in which:
        globals()[w]()
