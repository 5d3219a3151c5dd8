"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): native index build, pruned + exhaustive RayCast (mma.sync and
tcgen05 screens), traversal (hash tables, level driver), owner-shard ops on
one rank, MC with face-table re-reduction, HMC, verify_mesh."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

rng = np.random.default_rng(0)
for d, n in ((3, 600), (6, 3000)):
    pts = rng.random((n, d))
    ns = vb.NodeSet(pts)
    g = rng.integers(0, n, 2000).astype(np.int32)
    u = rng.standard_normal((2000, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    a = vb.raycast_batch(ns, pts[g], u, g[:, None], mode="pruned")
    b = vb.raycast_batch(ns, pts[g], u, g[:, None], mode="exhaustive")
    assert torch.equal(a.idx, b.idx)
    mesh = vb.voronoi_graph(ns, seed=0)
    rep = vb.verify_mesh(mesh, oracle=False)
    assert rep.passed, rep
    cells = np.array(mesh.bounded_cells()[:30], dtype=np.int32)
    mc = vb.mc_cells(ns, cells, 300, seed=1, max_faces=4)
    h = vb.hmc_cells(mesh, mc)
    loc = vb.voronoi_local(ns, rng.choice(n, 20, replace=False), hops=2)
    print(d, mesh.n_vertices, loc.n_vertices, float(h.volume.sum()), flush=True)
torch.cuda.synchronize()
print("sanitize workload done")
