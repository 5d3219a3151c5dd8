"""tcgen05 screen (VR_MMA=2) vs the exhaustive fp64 kernel: bitwise results
over d = 5..8, then config-2 kernel time.  Run once per VR_MMA value."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_10050_b200 as vb  # noqa: E402

mode = os.environ.get("VR_MMA", "1")
bad = 0
for d, n, m in ((5, 20000, 50000), (6, 30000, 80000), (7, 20000, 30000), (8, 50000, 30000)):
    pts = np.random.default_rng(d).random((n, d))
    ns = vb.NodeSet(pts)
    rng = np.random.default_rng(d + 100)
    g = rng.integers(0, n, m).astype(np.int32)
    u = rng.standard_normal((m, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    a = vb.raycast_batch(ns, pts[g], u, g[:, None], mode="pruned")
    b = vb.raycast_batch(ns, pts[g], u, g[:, None], mode="exhaustive", screen="fp64")
    ok = (torch.equal(a.idx, b.idx) and torch.equal(a.flag, b.flag) and
          torch.equal(torch.nan_to_num(a.t, 7.0), torch.nan_to_num(b.t, 7.0)))
    bad += not ok
    print(f"VR_MMA={mode} d={d}: pruned == exhaustive: {ok}", flush=True)
# config-2-shaped timing (random vertex-free rays from generators)
import bench  # noqa: E402
pts = bench.generators()
ns = vb.build_node_set(pts)
s, p, uu = bench.ray_recipe(10 ** 6)
need = np.unique(p)
sig, r = vb.descent_batch(ns, s[need], seed=0)
ps = np.zeros((bench.N_POOL, 7), dtype=np.int32)
pr = np.zeros((bench.N_POOL, 6))
ps[need], pr[need] = sig, r
x, u, g = bench.assemble(pts, ps, pr, p, uu)
xd, ud, gd = (torch.from_numpy(t).cuda() for t in (x, u, g))
work = torch.zeros(16, dtype=torch.int64, device="cuda")
for i in range(3):
    vb.raycast_batch(ns, xd, ud, gd, work=work if i == 0 else None)
ts = []
for i in range(5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    vb.raycast_batch(ns, xd, ud, gd, events=ev)
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
w = work.double().cpu().numpy()
print(f"VR_MMA={mode} config2 kernel ms: median {np.median(ts):.3f} all {np.round(ts, 3).tolist()}; "
      f"pairs/ray {w[0] / 1e6:.0f} node tests {w[5]:.0f} rare entries/ray {w[3] / 1e6:.2f}")
sys.exit(1 if bad else 0)
