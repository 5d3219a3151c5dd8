"""A/B timing of the config-5 local traversal (N=1e6, d=8, L=5 around 10k
seeds) and of the config-4 MC cells: min over repetitions, for comparing
library variants (VR_LIB_PATH) or VR_MMA settings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
ns.prune_index()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mesh, lv = vb.voronoi_local(ns, seeds, hops=5, return_levels=True)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    V = len(lv)
    del mesh, lv
    torch.cuda.empty_cache()
print(f"config5 L=5: min {min(ts):.3f} s  all {[round(t, 3) for t in ts]}  V={V}")
pts4 = np.random.default_rng(0).random((100000, 4))
ns4 = vb.NodeSet(pts4)
ns4.prune_index()
cells = np.arange(100000)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = vb.mc_cells(ns4, cells, 1000, seed=0)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    del res
print(f"config4 MC: min {min(ts):.3f} s  all {[round(t, 3) for t in ts]}")
