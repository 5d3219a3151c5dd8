"""Config-5 dense-level coherence: edge rays of a sample of the level-4
vertices of the 10,000-seed traversal (the rays of the dominant last level):
tiles visited per 32-ray warp by the pruned kernel vs the union of the rays'
FINAL spheres per 32 rays in the processing order, and per-ray need."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.raycast import coherent_order  # noqa: E402
from tools.coherence_study import need_mask  # noqa: E402


def main(frac=0.25):
    dev = torch.device("cuda", 0)
    d = 8
    pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    ns = vb.NodeSet(pts)
    seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
    mesh, lv = vb.voronoi_local(ns, seeds, hops=4, return_levels=True)
    dv = mesh.device_arrays()
    sel = np.nonzero(lv == 4)[0]
    sel = np.sort(np.random.default_rng(2).choice(sel, int(frac * len(sel)), replace=False))
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
    n = x.shape[0]
    work = torch.zeros(16, dtype=torch.int64, device=dev)
    res = vb.raycast_batch(ns, x, uu, eta, work=work, want_rp=False)
    w = work.double().cpu().numpy()
    nw = (n + 31) // 32
    print(f"rays {n} ({frac:.2f} of the level-4 vertices x {d + 1} edges)")
    print(f"kernel: tiles per warp {w[0] / (64 * 32) / nw:.1f}, node tests per warp {w[5] / nw:.0f}, "
          f"rare entries per ray {w[3] / n:.2f}")
    t = res.t.clone()
    t[~torch.isfinite(t)] = 1e3
    ix = ns.prune_index()
    X = torch.from_numpy(pts).to(dev)
    g = eta[:, 0].to(torch.int64)
    o = coherent_order(ix, eta, uu).to(torch.int64)
    CH = 1024
    tot = {gs: 0.0 for gs in (128, 32, 16, 8, 1)}
    starts = np.linspace(0, n - CH, 64).astype(np.int64) // 32 * 32
    for lo in starts:
        s_ = o[lo:lo + CH]
        m = need_mask(ix, x[s_], uu[s_], g[s_], t[s_], X, d)
        for gs in tot:
            tot[gs] += m.view(-1, gs, m.shape[1]).any(1).sum().item()
    for gs, v in tot.items():
        print(f"final-sphere union, groups of {gs:3d}: {v / (64 * CH / gs):7.1f} tiles per group "
              f"({v / (64 * CH):.2f} per ray)")


if __name__ == "__main__":
    main()
