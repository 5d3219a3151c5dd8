"""Host-side profile of the config-1 full diagram (latency-bound levels)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

ns = vb.build_node_set(np.random.default_rng(0).random((1000, 3)))
for _ in range(3):
    vb.voronoi_graph(ns, seed=0)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    vb.voronoi_graph(ns, seed=0)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
