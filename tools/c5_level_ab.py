"""Pruned-kernel time on config-5 dense-level edge rays (edges of half the
level-4 vertices; production order), median of 3 event-timed launches, plus
work counters -- A/B of library variants via VR_LIB_PATH."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

dev = torch.device("cuda", 0)
d = 8
pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
mesh, lv = vb.voronoi_local(ns, seeds, hops=4, return_levels=True)
dv = mesh.device_arrays()
sel = np.nonzero(lv == 4)[0]
sel = np.sort(np.random.default_rng(2).choice(sel, len(sel) // 2, replace=False))
sd = dv["sigma"][torch.as_tensor(sel, device=dev)]
rd = dv["r"][torch.as_tensor(sel, device=dev)]
u, ok = vb.vertex_directions_batch(ns, sd)
nv = sd.shape[0]
x = rd.repeat_interleave(d + 1, 0)
uu = u.reshape(-1, d)
keep = torch.ones((d + 1, d + 1), dtype=torch.bool, device=dev) ^ torch.eye(d + 1, dtype=torch.bool, device=dev)
eta = sd[:, None, :].expand(nv, d + 1, d + 1)[:, keep].reshape(nv * (d + 1), d).contiguous()
okf = ok.reshape(-1).bool()
x, uu, eta = x[okf].contiguous(), uu[okf].contiguous(), eta[okf].contiguous()
del mesh, dv
torch.cuda.empty_cache()
n = x.shape[0]
ts = []
for i in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    w = torch.zeros(16, dtype=torch.int64, device=dev)
    res = vb.raycast_batch(ns, x, uu, eta, want_rp=False, events=ev, work=w)
    torch.cuda.synchronize()
    if i:
        ts.append(ev[0].elapsed_time(ev[1]))
wk = w.double().cpu().numpy()
dig = int(res.idx.to(torch.int64).sum().item())
print(f"{os.path.basename(os.environ.get('VR_LIB_PATH', 'default'))}: rays {n} kernel {np.median(ts):.2f} ms "
      f"({[round(t, 1) for t in ts]}) tiles/warp {wk[0] / 2048 / (n / 32):.1f} node tests/warp "
      f"{wk[5] / (n / 32):.0f} entries/ray {wk[3] / n:.2f} idx-sum {dig}", flush=True)
