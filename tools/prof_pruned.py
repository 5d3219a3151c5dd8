"""Profiling driver for the pruned RayCast (config-2 generator-start rays)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
pts = np.random.default_rng(0).random((20000, 6))
ns = vb.NodeSet(pts)
ns.prune_index()
rng = np.random.default_rng(3)
g = rng.integers(0, 20000, n).astype(np.int32)
u = rng.standard_normal((n, 6))
u /= np.linalg.norm(u, axis=1, keepdims=True)
dev = torch.device("cuda", 0)
x, ud, gd = (torch.from_numpy(a).to(dev) for a in (pts[g], u, g[:, None].copy()))
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
vb.raycast_batch(ns, x, ud, gd, mode="pruned", events=e)
torch.cuda.synchronize()
print(f"pruned kernel_ms={e[0].elapsed_time(e[1]):.3f}")
