"""Config-5 local traversal (N=1e6, d=8, L=5 around 10k seeds): three timed
passes with the library / environment in effect (A/B via VR_LIB_PATH)."""
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
ts = []
for rep in range(4):
    st = vb.RaycastStats()
    work = torch.zeros(16, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mesh = vb.voronoi_local(ns, seeds, hops=5, stats=st, work=work)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    del mesh
print(f"{os.path.basename(os.environ.get('VR_LIB_PATH', 'default'))}: raycasts {st.raycasts} pairs "
      f"{int(work[0]) / 1e9:.1f} G times {[round(t, 3) for t in ts]}", flush=True)
