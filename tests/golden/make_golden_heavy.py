"""Generate the slow golden fixtures by running the UNMODIFIED reference.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src). Outputs land next to this script and are committed.

    python tests/golden/make_golden_heavy.py config3      # ~13 min, 1 core
    python tests/golden/make_golden_heavy.py config4exact # ~15 min, 1 core

config3:      voronoi_graph on SURVEY.md §8(d) config 3 (N=10,000, d=5,
              default_rng(0).standard_normal) -> sha256 digests of the sorted
              sigma array and of the sorted boundary-sigma multiset, counts.
config4exact: exact cell volumes (integrate_cell_poly) for the 2,000
              generators nearest (0.5,)^4 of config 4, from a certified
              12,000-point central sub-diagram (SURVEY.md §8(d) notes).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

import voronray as vr  # noqa: E402
from voronray.core import Mesh  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<i4").tobytes()).hexdigest()


def config3():
    pts = np.random.default_rng(0).standard_normal((10000, 5))
    t0 = time.time()
    stats = vr.RaycastStats()
    mesh = vr.voronoi_graph(vr.build_node_set(pts), seed=0, stats=stats)
    wall = time.time() - t0
    sig = np.array(sorted(mesh.vertices), dtype=np.int32)
    bnd = np.array(sorted(b.sigma for b in mesh.boundary), dtype=np.int32)
    n_int = sum(1 for c in mesh.edge_counts.values() if c == 2)
    out = {
        "config": "N=10000 d=5 default_rng(0).standard_normal, voronoi_graph(seed=0)",
        "input_sha16": hashlib.sha256(pts.tobytes()).hexdigest()[:16],
        "n_vertices": int(sig.shape[0]),
        "sigma_digest": digest(sig),
        "n_boundary": int(bnd.shape[0]),
        "boundary_digest": digest(bnd),
        "n_edges": len(mesh.edge_counts),
        "n_interior_edges": n_int,
        "raycasts": stats.raycasts,
        "nn_calls": stats.nn_calls,
        "reference_wall_s_1core": wall,
    }
    with open(os.path.join(HERE, "config3_reference.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(out)


def config4exact(n_sub=2000, n_ring=12000):
    pts = np.random.default_rng(0).random((100000, 4))
    full = vr.build_node_set(pts)
    order = np.argsort(np.linalg.norm(pts - 0.5, axis=1), kind="stable")
    ring = order[:n_ring]
    t0 = time.time()
    sub_ns = vr.NodeSet(pts[ring])
    sub = vr.voronoi_graph(sub_ns, seed=0)
    t_mesh = time.time() - t0
    shim = Mesh(full, {}, {}, [])
    vols = np.full(n_sub, np.nan)
    cert = np.zeros(n_sub, dtype=bool)
    t1 = time.time()
    for c in range(n_sub):
        ok = c not in sub.unbounded_cells() and len(sub.cell_vertices(c)) > 0
        if ok:
            for v in sub.cell_vertices(c):
                gsig = tuple(sorted(int(ring[s]) for s in v.sigma))
                if not vr.verify_vertex(shim, vr.VertexRecord(gsig, v.r)):
                    ok = False
                    break
        cert[c] = ok
        if ok:
            vols[c] = vr.integrate_cell_poly(sub, c, lambda x: 0.0).volume
    t_cert = time.time() - t1
    np.savez_compressed(os.path.join(HERE, "config4_exact.npz"),
                        cells=ring[:n_sub].astype(np.int64), volume=vols,
                        certified=cert)
    print({"certified": int(cert.sum()), "t_mesh": t_mesh, "t_cert": t_cert,
           "median_vol": float(np.nanmedian(vols))})


if __name__ == "__main__":
    {"config3": config3, "config4exact": config4exact}[sys.argv[1]]()
