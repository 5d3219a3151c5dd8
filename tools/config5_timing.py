"""Config 5: N=1e6, d=8 (fp32-upcast uniform); local traversal (all vertices
within L hops of the descent vertices of 10,000 random generators) and a
batched generator-start RayCast.  Reports phases and vertices/s."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

hops = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nseeds = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
t0 = time.perf_counter()
ns.prune_index()
ns.screen32()
torch.cuda.synchronize()
print(f"index build {time.perf_counter() - t0:.2f} s", flush=True)
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)[:nseeds]
t0 = time.perf_counter()
sig, r = vb.descent_batch(ns, seeds, seed=0)
print(f"descent {nseeds} seeds: {time.perf_counter() - t0:.2f} s", flush=True)
st = vb.RaycastStats()
torch.cuda.synchronize()
t0 = time.perf_counter()
mesh, lv = vb.voronoi_local(ns, seeds, hops=hops, stats=st, return_levels=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
V = len(lv)
print(f"local traversal L={hops}: {dt:.2f} s (incl. descent) V={V} "
      f"per-level={np.bincount(lv).tolist()} raycasts={st.raycasts} "
      f"-> {V / dt:.3e} vertices/s, {st.raycasts / dt:.3e} rays/s", flush=True)
