import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2405_10050_b200 as vb
pts5 = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns5 = vb.NodeSet(pts5); ns5.prune_index()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
st = vb.RaycastStats()
w = torch.zeros(16, dtype=torch.int64, device="cuda")
m, lv = vb.voronoi_local(ns5, seeds, hops=5, stats=st, return_levels=True, work=w)
torch.cuda.synchronize()
wk = w.double().cpu().numpy()
R = st.raycasts
print("rays", R, "pairs/ray", wk[0]/R, "tiles/warp", wk[0]/2048/(R/32), "node tests/warp", wk[5]/(R/32),
      "rare blocks/warp", wk[1]/(R/32), "rare iters/warp", wk[2]/(R/32), "entries/ray", wk[3]/R, "updates/ray", wk[4]/R)
