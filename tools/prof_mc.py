"""Profiling driver: config 4 MC (N=1e5, d=4, 1000 rays per cell) on the
first `cells` cells (k_mc_dirs, pruned RayCast, k_mc_reduce)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
pts = np.random.default_rng(0).random((100000, 4))
ns = vb.NodeSet(pts)
ns.prune_index()
for _ in range(2):
    res = vb.mc_cells(ns, np.arange(cells), 1000, seed=0)
    torch.cuda.synchronize()
print("ok", int((res.status == 0).sum()))
