import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2405_10050_b200 as vb
pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
ns.prune_index()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
mesh, lv = vb.voronoi_local(ns, seeds, hops=5, return_levels=True)
torch.cuda.synchronize()
print("V", len(lv))
