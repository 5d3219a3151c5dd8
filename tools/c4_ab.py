"""Config-4 MC (1e5 cells x 1000 Philox rays, d=4): median time of 3 passes,
pruned-kernel work counters and a volume checksum (A/B of VR_LIB_PATH)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

pts = np.random.default_rng(0).random((100000, 4))
ns = vb.NodeSet(pts)
ns.prune_index()
vb.mc_cells(ns, np.arange(2000), 1000, seed=0)
ts = []
for rep in range(4):
    w = torch.zeros(16, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = vb.mc_cells(ns, np.arange(100000), 1000, seed=0, work=w)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
wk = w.double().cpu().numpy()
R = 1e8
vol = np.asarray(res.volume, dtype=np.float64)
print(f"{os.path.basename(os.environ.get('VR_LIB_PATH', 'default'))}: {np.median(ts[1:]) * 1e3:.1f} ms "
      f"pairs/ray {wk[0] / R:.0f} tiles/warp {wk[0] / 2048 / (R / 32):.1f} node tests/warp "
      f"{wk[5] / (R / 32):.0f} entries/ray {wk[3] / R:.2f} vol-sum {np.nansum(vol):.15e}", flush=True)
