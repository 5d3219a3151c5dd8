"""One pruned RayCast launch over config-5 dense-level edge rays (the edges
of a quarter of the level-4 vertices of the 10k-seed traversal), inside the
NVTX range "target" -- for ncu --nvtx --nvtx-include "target/"."""
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
sel = np.sort(np.random.default_rng(2).choice(sel, len(sel) // 4, replace=False))
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
vb.raycast_batch(ns, x, uu, eta, want_rp=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("target")
vb.raycast_batch(ns, x, uu, eta, want_rp=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("rays", x.shape[0])
