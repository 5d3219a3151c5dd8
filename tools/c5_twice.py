import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2405_10050_b200 as vb
pts5 = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns5 = vb.NodeSet(pts5)
ns5.prune_index()
ns5.screen32()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
for rep in range(2):
    st = vb.RaycastStats()
    w5 = torch.zeros(16, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m5, lv = vb.voronoi_local(ns5, seeds, hops=5, stats=st, return_levels=True, work=w5)
    torch.cuda.synchronize()
    print(rep, time.perf_counter() - t0, len(lv), flush=True)
    if rep == 0:
        del m5, lv
