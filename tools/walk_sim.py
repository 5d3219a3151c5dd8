"""Per-ray walk study on config-5 dense-level edge rays (N=1e6, d=8): tiles
screened and node tests per ray for one ray walking the binary kd tree alone
(tools/walk_sim.c, exact fp64), under child orders x seeds x the lower-bound
prune.  Answers: is the kernel's tile count a warp-union effect or a per-ray
convergence effect?"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def lib():
    so = "/tmp/walk_sim.so"
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", so,
                           os.path.join(HERE, "walk_sim.c"), "-lm"])
    return ctypes.CDLL(so)


def P(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def main(nray=int(os.environ.get("NRAY", "1500"))):
    dev = torch.device("cuda", 0)
    d = int(os.environ.get("D", "8"))
    if d == 8:
        pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
        hops = 4
    else:  # config 2 (d = 6)
        pts = np.random.default_rng(0).random((20000, 6))
        hops = 3
    ns = vb.NodeSet(pts)
    seeds = np.random.default_rng(1).choice(len(pts), min(10000, len(pts) // 2), replace=False)
    mesh, lv = vb.voronoi_local(ns, seeds, hops=hops, return_levels=True)
    dv = mesh.device_arrays()
    sel = np.nonzero(lv == hops)[0]
    sel = np.sort(np.random.default_rng(2).choice(sel, nray // (d + 1) + 1, replace=False))
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
    res = vb.raycast_batch(ns, x, uu, eta, want_rp=False)
    ix = ns.prune_index()
    n = x.shape[0]
    X = torch.from_numpy(pts).to(dev)
    g = eta[:, 0].long()
    thr = (X[eta.long()] * uu[:, None]).sum(2).max(1).values
    thr = thr + 1e-12 * thr.abs().clamp(min=1.0)  # raycast.py:110-117 slack
    r02 = ((x - X[g]) ** 2).sum(1)
    s = (uu * X[g]).sum(1)
    inv = ix.inv_perm.long()
    PT = 64
    start = (inv[g] // PT)
    seeds_eta = (inv[eta.long()] // PT)
    # distinct eta tiles, -1 padded
    se = seeds_eta.cpu().numpy()
    se_u = np.full_like(se, -1)
    for k in range(n):
        u_ = np.unique(se[k])
        se_u[k, :len(u_)] = u_
    c = lambda a: np.ascontiguousarray(a.cpu().numpy())  # noqa: E731
    nb = c(ix.node_box)
    nr = c(ix.node_range)
    rec = c(ix.rec)
    xs, us, ths, r0s, ss, st = c(x), c(uu), c(thr), c(r02), c(s), c(start)
    tfin = c(res.t)
    ifin = c(res.idx)
    W = lib()
    W.walk_batch.restype = ctypes.c_int
    W.walk_batch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                             ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 7 + \
        [ctypes.c_int, ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4
    perm = c(ix.perm)
    print(f"d={d} n_tiles {ix.n_tiles} rays {n}", flush=True)

    def run(order, seedmode, lb):
        W.set_lb(lb)
        ot = np.zeros(n, np.int64)
        oq = np.zeros(n, np.int64)
        oi = np.zeros(n, np.int32)
        otb = np.zeros(n, np.float64)
        tb0 = None
        sdt, nsd = None, 0
        if seedmode == "own":
            sdt, nsd = np.ascontiguousarray(st[:, None]), 1
        elif seedmode == "eta":
            sdt, nsd = np.ascontiguousarray(se_u), se_u.shape[1]
        elif seedmode == "oracle":
            tb0 = np.where(np.isfinite(tfin), tfin * (1 + 1e-12), np.inf)
        rc = W.walk_batch(d, PT, ix.n_nodes, ix.n_tiles, P(nb), P(nr), P(rec), rec.shape[1],
                          rec.shape[0], n, P(xs), P(us), P(ths), P(r0s), P(ss), P(st), P(sdt),
                          nsd, P(tb0), order, P(ot), P(oq), P(oi), P(otb))
        assert rc == 0
        idx = np.where(oi >= 0, perm[np.maximum(oi, 0)], -1)
        agree = np.mean((idx == ifin) | (seedmode == "oracle"))
        return ot.mean(), oq.mean(), agree

    names = {0: "start-tile child first", 1: "nearest (d2) first", 2: "lower bound first (DFS)",
             3: "best-first (LB heap)"}
    W.get_sub_needed.restype = ctypes.c_int64
    W.get_sub_needed_sph.restype = ctypes.c_int64
    W.set_joint(0)

    def kd_within_tiles(rec, levels):
        """rows of each 64-row tile re-ordered by `levels` median splits on
        the widest dimension (sub-boxes of 64 >> levels rows)"""
        rows = rec.reshape(-1, PT, rec.shape[1]).copy()
        for lv in range(levels):
            g = 1 << lv
            blk = rows.reshape(rows.shape[0] * g, PT // g, rows.shape[2])
            xs_ = np.where(np.isinf(blk[:, :, d:d + 1]), np.nan, blk[:, :, :d])
            ext = np.nanmax(xs_, 1) - np.nanmin(xs_, 1)
            ax = np.nan_to_num(ext, nan=-1).argmax(1)
            key = np.take_along_axis(np.nan_to_num(xs_, nan=np.inf), ax[:, None, None], 2)[:, :, 0]
            o = np.argsort(key, 1, kind="stable")
            blk = np.take_along_axis(blk, o[:, :, None], 1)
            rows = blk.reshape(rows.shape)
        return np.ascontiguousarray(rows.reshape(rec.shape))

    rec_orig = rec
    for tag, rr in (("tile row order", rec_orig), ("kd within tiles", kd_within_tiles(rec_orig, 3))):
        rec = rr
        for sub in (32, 16, 8):
            W.set_sub(sub)
            tl, ts, ag = run(0, "oracle", 1)
            print(f"{tag}: oracle seed, {sub}-row sub-boxes: tiles/ray {tl:.2f} -> pairs/ray "
                  f"{64 * tl:.0f}; needed sub-boxes/ray {W.get_sub_needed() / n:.2f} -> pairs/ray "
                  f"{sub * W.get_sub_needed() / n:.0f}; with bounding spheres "
                  f"{W.get_sub_needed_sph() / n:.2f} -> {sub * W.get_sub_needed_sph() / n:.0f}", flush=True)
    rec = rec_orig
    W.set_sub(0)
    for seedmode in ("oracle", "own"):
      for joint in (0,):
        W.set_joint(joint)
        print(f"joint box/halfspace/sphere test: {joint}")
        for lb in (1,):
            for order in (0, 1, 3):
                tl, ts, ag = run(order, seedmode, lb)
                print(f"seed={seedmode:6s} lb_prune={lb} {names[order]:26s} tiles/ray {tl:7.2f} "
                      f"node tests/ray {ts:8.1f} agree {ag:.4f}", flush=True)


if __name__ == "__main__":
    main()
