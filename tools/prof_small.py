"""One config-1 traversal for profiling the persistent small-level kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_10050_b200 as vb
ns = vb.build_node_set(np.random.default_rng(0).random((1000, 3)))
for _ in range(3):
    vb.voronoi_graph(ns, seed=0)
torch.cuda.synchronize()
