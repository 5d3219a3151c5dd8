"""How many generator tiles does a warp of 32 rays need, for different ray
orders?  Lower bound per ray = tiles whose box meets the FINAL incircle
sphere and the forward halfspace (the pruned kernel, whose spheres shrink
over time, screens at least this union).  Config-2 rays.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.raycast import coherent_order, direction_bucket  # noqa: E402


def need_mask(ix, x, u, g, t, X, d):
    nt = ix.tile_box.shape[0]
    lo, hi = ix.tile_box[:, :d], ix.tile_box[:, d:]
    z = x + t[:, None] * u
    rho2 = ((z - X[g]) ** 2).sum(1)
    thr = (u * X[g]).sum(1)
    e = torch.clamp(torch.maximum(lo[None] - z[:, None], z[:, None] - hi[None]), min=0)
    d2 = (e * e).sum(2)
    umax = torch.where(u[:, None] > 0, u[:, None] * hi[None], u[:, None] * lo[None]).sum(2)
    return (d2 < rho2[:, None]) & (umax > thr[:, None])


def main():
    dev = torch.device("cuda", 0)
    pts = np.random.default_rng(0).random((20000, 6))
    d = 6
    ns = vb.NodeSet(pts)
    rng = np.random.default_rng(3)
    n = 1_000_000
    u = rng.standard_normal((n, 6))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    s = np.random.default_rng(1).choice(20000, 10000, replace=False)
    sig, r = vb.descent_batch(ns, s, seed=0)
    p = np.random.default_rng(2).integers(0, 10000, n)
    x = r[p]
    sg = sig[p]
    proj = np.einsum("kd,ksd->ks", u, pts[sg])
    g = sg[np.arange(n), np.argmax(proj, 1)].astype(np.int32)
    xd, ud, gd = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, u, g))
    res = vb.raycast_batch(ns, xd, ud, gd[:, None])
    t = res.t.clone()
    t[~torch.isfinite(t)] = 1e3
    ix = ns.prune_index()
    X = torch.from_numpy(pts).to(dev)
    gl = gd.to(torch.int64)
    pos = ix.inv_perm.to(torch.int64)
    hit = res.idx.to(torch.int64).clamp(min=0)
    # seed prediction: best candidate of the start tile
    PT = 64
    st = pos[gl] // PT
    cand = ix.perm.to(torch.int64)[(st[:, None] * PT + torch.arange(PT, device=dev)).clamp(max=ns.n - 1)]
    Xc = X[cand]
    q = (Xc * ud[:, None]).sum(2)
    s0 = (ud * X[gl]).sum(1)
    aa = ((xd[:, None] - Xc) ** 2).sum(2)
    base = ((xd - X[gl]) ** 2).sum(1)
    tt = (aa - base[:, None]) / (2 * (q - s0[:, None]))
    tt = torch.where(q > s0[:, None] + 1e-12, tt, torch.full_like(tt, float("inf")))
    sb = cand[torch.arange(n, device=dev), tt.argmin(1)]
    tseed = tt.min(1).values
    zs = xd + torch.where(torch.isfinite(tseed), tseed, torch.zeros_like(tseed))[:, None] * ud
    bucket = direction_bucket(ud)

    def zkey(z):
        # kd tile of the nearest generator of z, approximated by morton-like
        # quantisation of z (8 bins / axis)
        qz = ((z - X.min(0).values) / (X.max(0).values - X.min(0).values) * 8).clamp(0, 7).to(torch.int64)
        k = torch.zeros(z.shape[0], dtype=torch.int64, device=dev)
        for b in range(3):
            for a in range(d):
                k = (k << 1) | ((qz[:, a] >> (2 - b)) & 1)
        return k

    orders = {
        "input order": torch.arange(n, device=dev),
        "coherent (pos g, bucket)": coherent_order(ix, gd[:, None], ud).to(torch.int64),
        "pos g only": torch.sort(pos[gl], stable=True).indices,
        "vertex id (p), bucket": torch.sort(torch.from_numpy(p).to(dev) * 256 + bucket, stable=True).indices,
        "pos seed hit": torch.sort(pos[sb] * 1_000_000 + pos[gl], stable=True).indices,
        "pos seed hit, bucket": torch.sort(pos[sb] * 256 + bucket, stable=True).indices,
        "morton seed vertex": torch.sort(zkey(zs), stable=True).indices,
        "pos final hit (ideal)": torch.sort(pos[hit] * 1_000_000 + pos[gl], stable=True).indices,
        "morton final vertex (ideal)": torch.sort(zkey(xd + t[:, None] * ud), stable=True).indices,
    }
    nw = n // 32
    per_ray = 0.0
    acc = {k: 0.0 for k in orders}
    CH = 32768
    t0 = time.time()
    inv = {k: torch.empty_like(o) for k, o in orders.items()}
    for k, o in orders.items():
        inv[k][o] = torch.arange(n, device=dev)
    for lo in range(0, n, CH):
        pass
    # evaluate union per warp: process warps in chunks
    for k, o in orders.items():
        tot = 0
        for lo in range(0, n, CH):
            sel = o[lo:lo + CH]
            m = need_mask(ix, xd[sel], ud[sel], gl[sel], t[sel], X, d)
            if k == "input order":
                per_ray += m.sum().item()
            w = m.view(-1, 32, m.shape[1]).any(1)
            tot += w.sum().item()
        acc[k] = tot / nw
    o = orders["coherent (pos g, bucket)"]
    per_warp = []
    for lo in range(0, n, CH):
        sel = o[lo:lo + CH]
        m = need_mask(ix, xd[sel], ud[sel], gl[sel], t[sel], X, d)
        per_warp.append(m.view(-1, 32, m.shape[1]).any(1).sum(1).cpu())
    pw = torch.cat(per_warp).numpy()
    print("union tiles per warp (coherent order): mean %.1f p50 %d p99 %d p99.9 %d max %d; "
          "warps > 150 tiles: %d" % (pw.mean(), np.percentile(pw, 50), np.percentile(pw, 99),
                                     np.percentile(pw, 99.9), pw.max(), (pw > 150).sum()))
    # union with the SEED spheres (best candidate of the start tile), i.e. a
    # tile list fixed before any screening
    ts = torch.where(torch.isfinite(tseed), tseed, torch.full_like(tseed, 1e3))
    tot_s = per_s = 0
    for lo in range(0, n, CH):
        sel = o[lo:lo + CH]
        m = need_mask(ix, xd[sel], ud[sel], gl[sel], ts[sel], X, d)
        per_s += m.sum().item()
        tot_s += m.view(-1, 32, m.shape[1]).any(1).sum().item()
    print(f"  seed spheres: per-ray need {per_s / n:.1f} tiles, warp union {tot_s / nw:.1f} tiles")
    # outliers: union without the k rays of largest individual need
    for kx in (1, 2, 4, 8):
        tot_u = 0
        for lo in range(0, n, CH):
            sel = o[lo:lo + CH]
            m = need_mask(ix, xd[sel], ud[sel], gl[sel], t[sel], X, d).view(-1, 32, ix.tile_box.shape[0])
            need = m.sum(2)                                   # (warps, 32)
            drop = need.topk(kx, dim=1).indices               # (warps, kx)
            keep = torch.ones_like(need, dtype=torch.bool).scatter_(1, drop, False)
            tot_u += (m & keep[:, :, None]).any(1).sum().item()
        print(f"  union without the {kx} largest rays per warp: {tot_u / nw:.1f} tiles")
    esc = ~torch.isfinite(res.t)
    print("escaped rays", int(esc.sum()), "warps with an escaped ray",
          int(esc[o].view(-1, 32).any(1).sum()))
    for gs in (16, 8, 4, 2):
        tot_max = tot_mean = 0
        for lo in range(0, n, CH):
            sel = o[lo:lo + CH]
            m = need_mask(ix, xd[sel], ud[sel], gl[sel], t[sel], X, d)
            w = m.view(-1, 32 // gs, gs, m.shape[1]).any(2).sum(2)  # (warps, groups)
            tot_max += w.max(1).values.sum().item()
            tot_mean += w.float().mean(1).sum().item()
        print(f"  groups of {gs:2d} rays: union tiles/group {tot_mean / nw:7.2f}, "
              f"max over the warp's groups {tot_max / nw:7.2f}")
    for gsz in (64, 128):  # larger groups (2 / 4 rays per lane, or CTA-wide)
        tot_g = 0
        for lo in range(0, n, CH):
            sel = o[lo:lo + CH]
            m = need_mask(ix, xd[sel], ud[sel], gl[sel], t[sel], X, d)
            tot_g += m.view(-1, gsz, m.shape[1]).any(1).sum().item()
        print(f"  groups of {gsz:3d} rays: union tiles/group {tot_g / (n // gsz):7.2f} "
              f"({tot_g / (n // gsz) / gsz:.3f} per ray)")
    print(f"tiles total {ix.tile_box.shape[0]}; per-ray need (final sphere) {per_ray / n:.2f}")
    for k in orders:
        print(f"  {k:32s} union tiles/warp {acc[k]:7.2f}")
    print("study time", time.time() - t0)


if __name__ == "__main__":
    main()
