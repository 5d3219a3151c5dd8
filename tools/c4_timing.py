"""Config 4 (1e5 cells x 1000 Philox rays, d=4): MC volumes/areas timing."""
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
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = vb.mc_cells(ns, np.arange(100000), 1000, seed=0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"config4 MC: {dt:.3f} s  {1e8 / dt:.3e} rays/s  bounded={(res.status == 0).sum()}")
