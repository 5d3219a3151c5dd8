"""Host profile of a full-diagram traversal: config 3 (N=10,000, d=5,
Gaussian; default) or config 1 (argument "1": N=1,000, d=3, uniform):
per-level overhead of the level-synchronous traversal (after warm runs)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "1":
    pts = np.random.default_rng(0).random((1000, 3))
else:
    pts = np.random.default_rng(0).standard_normal((10000, 5))
ns = vb.NodeSet(pts)
ns.prune_index()
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = vb.voronoi_graph(ns, seed=0)
    torch.cuda.synchronize()
    print(f"run {i}: {time.perf_counter() - t0:.4f} s")
pr = cProfile.Profile()
pr.enable()
m = vb.voronoi_graph(ns, seed=0)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

# device-side kernel time of one run (CUPTI via torch.profiler): how much of
# the wall time is GPU work vs host overhead between launches
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m = vb.voronoi_graph(ns, seed=0)
    torch.cuda.synchronize()
tot = sum(e.device_time_total for e in prof.key_averages()) / 1e3
print(f"device kernel time {tot:.2f} ms")
print(prof.key_averages().table(sort_by="device_time_total", row_limit=12))
