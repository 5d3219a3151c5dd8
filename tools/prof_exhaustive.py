"""Profiling driver: the exhaustive fp64-screen RayCast on the config-2 rays
(every (ray, generator) pair screened; the FP64-pipe roofline reference)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_10050_b200 as vb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
screen = sys.argv[2] if len(sys.argv) > 2 else "fp64"
mode = sys.argv[3] if len(sys.argv) > 3 else "exhaustive"
pts = bench.generators()
ns = vb.NodeSet(pts)
s, p_all, u_all = bench.ray_recipe(n)
need = np.unique(p_all)
sig_n, r_n = vb.descent_batch(ns, s[need], seed=0)
pool_sig = np.zeros((bench.N_POOL, bench.DIM + 1), dtype=np.int32)
pool_r = np.zeros((bench.N_POOL, bench.DIM))
pool_sig[need], pool_r[need] = sig_n, r_n
x, u, g = bench.assemble(pts, pool_sig, pool_r, p_all, u_all)
xd, ud, gd = (torch.from_numpy(a).cuda() for a in (x, u, g))
for _ in range(2):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    vb.raycast_batch(ns, xd, ud, gd, mode=mode, screen=screen, events=e)
    torch.cuda.synchronize()
    print(f"{mode} {screen} kernel_ms={e[0].elapsed_time(e[1]):.3f} for {n} rays")
