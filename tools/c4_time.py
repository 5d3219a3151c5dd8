"""Config-4 MC (1e5 cells x 1000 rays, d=4): timed passes with the library in effect."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

pts4 = np.random.default_rng(0).random((100000, 4))
ns4 = vb.NodeSet(pts4)
ns4.prune_index()
cells = np.arange(100000)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = vb.mc_cells(ns4, cells, 1000, seed=0)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    vol = float(res.volume[:1000].sum()) if hasattr(res, "volume") else 0.0
    del res
print(f"{os.path.basename(os.environ.get('VR_LIB_PATH', 'default'))}: config4 MC times {[round(t, 4) for t in ts]} vol1000 {vol:.12g}")
