"""Config-5 edge rays (N=1e6, d=8): per-ray tile need (final sphere) vs the
union over groups of G consecutive rays in the kernel's processing order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.raycast import coherent_order  # noqa: E402
from tools.coherence_study import need_mask  # noqa: E402
from tools.sweep_pruned import edge_rays  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    ns = vb.NodeSet(pts)
    seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
    x, u, eta = edge_rays(ns, pts, seeds)
    xd, ud, ed = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, u, eta))
    res = vb.raycast_batch(ns, xd, ud, ed)
    t = res.t.clone()
    t[~torch.isfinite(t)] = 1e3
    ix = ns.prune_index()
    X = torch.from_numpy(pts).to(dev)
    g = ed[:, 0].to(torch.int64)
    o = coherent_order(ix, ed, ud).to(torch.int64)
    n = (xd.shape[0] // 32) * 32
    CH = 1024
    tot = {gs: 0.0 for gs in (32, 16, 8, 4, 1)}
    for lo in range(0, n, CH):
        sel = o[lo:min(lo + CH, n)]
        m = need_mask(ix, xd[sel], ud[sel], g[sel], t[sel], X, 8)
        for gs in tot:
            tot[gs] += m.view(-1, gs, m.shape[1]).any(1).sum().item() * gs / 32
    nw = n // 32
    for gs, v in tot.items():
        print(f"groups of {gs:2d} rays: tiles per warp-equivalent {v / nw:8.1f}  "
              f"(per group {v / nw * gs / 32:7.1f})")


if __name__ == "__main__":
    main()
