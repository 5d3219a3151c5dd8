"""cProfile of descent_batch on config 5's 10,000 starts (N=1e6, d=8)."""
import cProfile
import os
import pstats
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
vb.descent_batch(ns, seeds, seed=0)
torch.cuda.synchronize()
t0 = time.perf_counter()
vb.descent_batch(ns, seeds, seed=0)
torch.cuda.synchronize()
print("descent_batch", (time.perf_counter() - t0) * 1e3, "ms")
pr = cProfile.Profile()
pr.enable()
vb.descent_batch(ns, seeds, seed=0)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
