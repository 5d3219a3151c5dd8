"""Host profile of the config-5 local traversal (second run) and its device
kernel time (CUPTI via torch.profiler)."""
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
for i in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m, lv = vb.voronoi_local(ns, seeds, hops=5, return_levels=True)
    torch.cuda.synchronize()
    print(f"run {i}: {time.perf_counter() - t0:.3f} s")
    del m, lv
    torch.cuda.empty_cache()
pr = cProfile.Profile()
pr.enable()
m, lv = vb.voronoi_local(ns, seeds, hops=5, return_levels=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
del m, lv
torch.cuda.empty_cache()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m, lv = vb.voronoi_local(ns, seeds, hops=5, return_levels=True)
    torch.cuda.synchronize()
tot = sum(e.device_time_total for e in prof.key_averages()) / 1e3
print(f"device kernel time {tot:.1f} ms")
