"""Profiling driver: pruned RayCast on config 5 (N=1e6, d=8) generator-start rays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
ns.prune_index()
ns.screen32()
rng = np.random.default_rng(4)
g = rng.integers(0, 10 ** 6, n).astype(np.int32)
u = rng.standard_normal((n, 8))
u /= np.linalg.norm(u, axis=1, keepdims=True)
dev = torch.device("cuda", 0)
x, ud, gd = (torch.from_numpy(a).to(dev) for a in (pts[g], u, g[:, None].copy()))
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
vb.raycast_batch(ns, x, ud, gd, mode="pruned", events=e)
torch.cuda.synchronize()
print(f"c5 pruned kernel_ms={e[0].elapsed_time(e[1]):.3f}")
