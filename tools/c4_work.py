import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2405_10050_b200 as vb
pts = np.random.default_rng(0).random((100000, 4))
ns = vb.NodeSet(pts); ns.prune_index()
w = torch.zeros(16, dtype=torch.int64, device="cuda")
res = vb.mc_cells(ns, np.arange(100000), 1000, seed=0, work=w)
torch.cuda.synchronize()
wk = w.double().cpu().numpy(); R = 1e8
print("pairs/ray", wk[0]/R, "tiles/warp", wk[0]/2048/(R/32), "node tests/warp", wk[5]/(R/32),
      "rare blocks/warp", wk[1]/(R/32), "rare iters/warp", wk[2]/(R/32), "entries/ray", wk[3]/R, "updates/ray", wk[4]/R)
