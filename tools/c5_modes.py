"""Config-5 L=5 traversal time under the current VR_MMA / VR_COOP settings
(median of 3 passes after a warm one) and the pruned-kernel work counters."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
ns.prune_index()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
ts = []
for rep in range(4):
    w = torch.zeros(16, dtype=torch.int64, device="cuda")
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mesh, lv = vb.voronoi_local(ns, seeds, hops=5, return_levels=True, work=w)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    del mesh
wk = w.double().cpu().numpy()
print(f"VR_MMA={os.environ.get('VR_MMA', '-')} V={len(lv)} median {np.median(ts[1:]):.3f} s "
      f"passes {np.round(ts, 3).tolist()} pairs {wk[0]:.3e} node_tests {wk[5]:.3e} "
      f"rare_entries {wk[3]:.3e}")
