"""Config-3 full diagram (N=1e4, d=5): per-level frontier sizes and the median
time of 5 passes (run with VR_SMALL_LEVELS=0/1 to compare drivers)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_10050_b200 as vb
pts = np.random.default_rng(0).standard_normal((10000, 5))
ns = vb.build_node_set(pts)
ns.prune_index()
m, info = vb.voronoi_graph(ns, seed=0, return_info=True)
ts = []
for _ in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    vb.voronoi_graph(ns, seed=0)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
F = [a for a, b in info["levels"]]
print(f"VR_SMALL_LEVELS={os.environ.get('VR_SMALL_LEVELS', '-')}: median {np.median(ts[1:]) * 1e3:.2f} ms "
      f"levels {len(F)}; frontier sizes {F}")
