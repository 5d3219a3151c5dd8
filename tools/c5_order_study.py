"""Config-5 dense-level rays (N=1e6, d=8): pruned-kernel time and work per
processing order.  The rays are the edge rays of the level-4 vertices of the
10,000-seed traversal; every order is passed to vr_raycast_pruned directly.

Orders: the production one (kd position of eta[0], direction class), the
kd position of the seed hit (best candidate of the start tile: computable
before the RayCast), a Morton code of the seed vertex, and, as an ideal, the
kd position of the final hit / Morton code of the final vertex."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200 import _lib  # noqa: E402
from paper_2405_10050_b200.raycast import coherent_order, direction_bucket  # noqa: E402


def morton(z, lo, hi, bits=3):
    d = z.shape[1]
    q = ((z - lo) / (hi - lo) * (1 << bits)).clamp(0, (1 << bits) - 1).to(torch.int64)
    k = torch.zeros(z.shape[0], dtype=torch.int64, device=z.device)
    for b in range(bits):
        for a in range(d):
            k = (k << 1) | ((q[:, a] >> (bits - 1 - b)) & 1)
    return k


def main(frac=float(os.environ.get("FRAC", "0.5"))):
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
    del mesh, dv
    torch.cuda.empty_cache()
    n = x.shape[0]
    print(f"rays {n} (edges of {nv} level-4 vertices)", flush=True)
    ix = ns.prune_index()
    rec, sqmax = ns.device_records()
    s32 = ns.screen32(dev)
    L = _lib.lib()
    idx = torch.empty(n, dtype=torch.int32, device=dev)
    t = torch.empty(n, dtype=torch.float64, device=dev)
    flag = torch.empty(n, dtype=torch.uint8, device=dev)
    rl = torch.empty(n, dtype=torch.int32, device=dev)
    rc = torch.zeros(1, dtype=torch.int32, device=dev)

    def run(order, reps=3):
        ts = []
        for r in range(reps):
            w = torch.zeros(16, dtype=torch.int64, device=dev)
            rc.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            _lib.check(L.vr_raycast_pruned(_lib.ptr(rec), ns.n, d, sqmax, ctypes.byref(s32.struct),
                                           ctypes.byref(ix.struct), _lib.ptr(x), _lib.ptr(uu),
                                           _lib.ptr(eta), d, n, _lib.ptr(order), _lib.ptr(idx),
                                           _lib.ptr(t), None, _lib.ptr(flag), _lib.ptr(rl),
                                           _lib.ptr(rc), _lib.ptr(w), None), "pruned")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        wk = w.double().cpu().numpy()
        nw = n / 32
        return (np.median(ts), wk[0] / 2048 / nw, wk[5] / nw, wk[3] / n)

    o_cur = coherent_order(ix, eta, uu).to(torch.int32)
    ms, tpw, npw, ent = run(o_cur)
    print(f"{'production order':34s} {ms:8.2f} ms  tiles/warp {tpw:7.1f} node tests/warp {npw:7.0f} "
          f"rare entries/ray {ent:.2f}", flush=True)
    idx0, t0 = idx.clone(), t.clone()
    pos = ix.inv_perm.to(torch.int64)
    g = eta[:, 0].to(torch.int64)
    X = torch.from_numpy(pts).to(dev)
    # seed: best valid candidate of g's tile (fp64, torch, chunked)
    PT = 64
    sb = torch.empty(n, dtype=torch.int64, device=dev)
    tseed = torch.empty(n, dtype=torch.float64, device=dev)
    permL = ix.perm.to(torch.int64)
    CH = 1 << 18
    for lo in range(0, n, CH):
        hi = min(n, lo + CH)
        st = pos[g[lo:hi]] // PT
        cand = permL[(st[:, None] * PT + torch.arange(PT, device=dev)).clamp(max=ns.n - 1)]
        Xc = X[cand]
        xs, us = x[lo:hi], uu[lo:hi]
        q = (Xc * us[:, None]).sum(2)
        thr = (X[eta[lo:hi].to(torch.int64)] * us[:, None]).sum(2).max(1).values
        s0 = (us * X[g[lo:hi]]).sum(1)
        aa = ((xs[:, None] - Xc) ** 2).sum(2)
        base = ((xs - X[g[lo:hi]]) ** 2).sum(1)
        tt = (aa - base[:, None]) / (2 * (q - s0[:, None]))
        tt = torch.where(q > thr[:, None] + 1e-12, tt, torch.full_like(tt, float("inf")))
        m = tt.min(1)
        tseed[lo:hi] = m.values
        sb[lo:hi] = cand[torch.arange(hi - lo, device=dev), m.indices]
    fin = torch.isfinite(tseed)
    print(f"seed pass finite for {fin.double().mean().item():.3f} of rays; seed hit == final "
          f"{(sb == idx0.to(torch.int64)).double().mean().item():.3f}", flush=True)
    bucket = direction_bucket(uu)
    lo_, hi_ = X.min(0).values, X.max(0).values
    zs = x + torch.where(fin, tseed, torch.zeros_like(tseed))[:, None] * uu
    tf = torch.where(torch.isfinite(t0), t0, torch.zeros_like(t0))
    zf = x + tf[:, None] * uu
    hit = idx0.to(torch.int64).clamp(min=0)
    sbp = torch.where(fin, pos[sb], pos[g])
    orders = {
        "pos seed hit, bucket": sbp * 256 + bucket,
        "pos seed hit, pos g": sbp * (1 << 21) + pos[g],
        "morton seed vertex (3 bits)": morton(zs, lo_, hi_, 3),
        "morton seed vertex (2 bits)": morton(zs, lo_, hi_, 2) * 256 + bucket,
        "pos final hit, bucket (ideal)": pos[hit] * 256 + bucket,
        "morton final vertex (ideal)": morton(zf, lo_, hi_, 3),
    }
    for name, key in orders.items():
        o = torch.sort(key, stable=True).indices.to(torch.int32)
        ms, tpw, npw, ent = run(o)
        same = torch.equal(idx, idx0)
        print(f"{name:34s} {ms:8.2f} ms  tiles/warp {tpw:7.1f} node tests/warp {npw:7.0f} "
              f"rare entries/ray {ent:.2f}  same={same}", flush=True)
    os.environ["VR_COOP"] = "1"


if __name__ == "__main__":
    t_ = time.time()
    main()
    print("time", time.time() - t_)
