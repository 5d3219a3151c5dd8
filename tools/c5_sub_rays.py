"""Config-5 local traversal: edge raycasts and time per sub-round setting."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
ns.prune_index()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
for rays, mx in ((0, 1), (0, 1), (4000000, 2), (4000000, 4), (4000000, 8), (1000000, 16), (1000000, 64)):
    vb.set_sub_rounds(rays, mx)
    ts = []
    for rep in range(3):
        st = vb.RaycastStats()
        work = torch.zeros(16, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mesh = vb.voronoi_local(ns, seeds, hops=5, stats=st, work=work)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        nv = mesh.n_vertices if hasattr(mesh, "n_vertices") else -1
        del mesh
    print(f"sub_rays={rays} max={mx}: raycasts {st.raycasts} pairs {int(work[0]) / 1e9:.1f} G "
          f"times {[round(t, 3) for t in ts]}", flush=True)
