"""Profiling driver: one fused RayCast launch on config-2-shaped rays.

Generator-start rays (x = x_g, eta = (g,)) so no descent kernels run before
the profiled launch.  Usage (on the GPU box):
    ncu --set full --clock-control none --import-source on -k regex:k_raycast -c 1 \
        -o gpurun_out/prof python tools/prof_raycast.py [n_rays] [d] [n_gen]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 6
N = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
pts = np.random.default_rng(0).random((N, d))
ns = vb.NodeSet(pts)
rng = np.random.default_rng(3)
g = rng.integers(0, N, n).astype(np.int32)
u = rng.standard_normal((n, d))
u /= np.linalg.norm(u, axis=1, keepdims=True)
dev = torch.device("cuda", 0)
x = torch.from_numpy(pts[g]).to(dev)
ud = torch.from_numpy(u).to(dev)
gd = torch.from_numpy(g[:, None].copy()).to(dev)
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
res = vb.raycast_batch(ns, x, ud, gd, events=e)
torch.cuda.synchronize()
print(f"rays={n} d={d} N={N} kernel_ms={e[0].elapsed_time(e[1]):.3f} "
      f"recheck_ms={e[1].elapsed_time(e[2]):.3f} "
      f"rays/s={n / (e[0].elapsed_time(e[1]) * 1e-3):.3e}")
