"""Pruned vs exhaustive RayCast: kernel time, screened pairs, pair rate."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402


def run(name, ns, x, u, eta, modes=("exhaustive", "pruned")):
    dev = torch.device("cuda", 0)
    xd, ud, ed = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, u, eta))
    n = xd.shape[0]
    ns.prune_index()
    for mode in modes:
        work = torch.zeros(16, dtype=torch.int64, device=dev)
        vb.raycast_batch(ns, xd, ud, ed, mode=mode)  # warm
        ks = []
        for rep in range(int(os.environ.get("REPS", "5"))):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            work.zero_()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_push(f"sweep_{mode}")
            vb.raycast_batch(ns, xd, ud, ed, mode=mode, events=e, work=work)
            torch.cuda.nvtx.range_pop()
            torch.cuda.synchronize()
            ks.append(e[0].elapsed_time(e[1]))
        k = float(np.median(ks))
        if os.environ.get("CHECK") and mode == "pruned":
            ref = vb.raycast_batch(ns, xd, ud, ed, mode="exhaustive")
            got = vb.raycast_batch(ns, xd, ud, ed, mode="pruned")
            bad = ((ref.idx != got.idx) | (ref.flag != got.flag)).sum().item()
            print(f"   CHECK vs exhaustive: {bad} mismatching rays of {n}", flush=True)
        w = work.cpu().numpy()
        pairs = int(w[0]) if mode == "pruned" else n * ns.n
        if mode == "pruned":
            nw = (n + 31) // 32
            print(f"   per warp: rare blocks {w[1] / nw:.1f}, rare iterations {w[2] / nw:.1f}; "
                  f"per ray: entries {w[3] / n:.2f}, sphere updates {w[4] / n:.2f}; "
                  f"tiles/warp {w[0] / 2048 / nw:.1f}, node tests/warp {w[5] / nw:.1f}")
            if w[6:11].sum():
                print("   rare entries per ray: outside %.2f self %.2f behind %.2f band %.2f improving %.2f"
                      % tuple(w[6:11] / n))
        print(f"{name:28s} {mode:10s} rays={n:8d} kernel={k:8.3f} ms  rays/s={n / k * 1e3:9.3e}"
              f"  pairs/ray={pairs / n:9.1f}  Gpairs/s={pairs / k / 1e6:8.1f}", flush=True)


def edge_rays(ns, pts, seeds):
    """All d+1 edge rays of the descent vertices of `seeds` (traversal rays,
    |eta| = d, eta sorted so eta[0] is the smallest index)."""
    sig, r = vb.descent_batch(ns, seeds, seed=0)
    d = pts.shape[1]
    u, ok = vb.vertex_directions_batch(ns, sig)
    u = u.cpu().numpy().reshape(-1, d)
    ok = ok.cpu().numpy().reshape(-1).astype(bool)
    x = np.repeat(r, d + 1, axis=0)
    eta = np.stack([np.delete(s_, k) for s_ in sig for k in range(d + 1)]).astype(np.int32)
    eta.sort(axis=1)
    return x[ok], u[ok], eta[ok]



if __name__ == "__main__":
    which = sys.argv[1:] or ["c2gen", "c2vert", "c5gen", "c4mc"]
    if os.environ.get("MODES"):
        run.__defaults__ = (tuple(os.environ["MODES"].split(",")),)
    if "c2gen" in which or "c2vert" in which:
        pts = np.random.default_rng(0).random((20000, 6))
        ns = vb.NodeSet(pts)
        rng = np.random.default_rng(3)
        n = 1_000_000
        u = rng.standard_normal((n, 6))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        if "c2gen" in which:
            g = rng.integers(0, 20000, n).astype(np.int32)
            run("c2 generator-start", ns, pts[g], u, g[:, None])
        if "c2vert" in which:
            s = np.random.default_rng(1).choice(20000, 10000, replace=False)
            t0 = time.time()
            sig, r = vb.descent_batch(ns, s, seed=0)
            print("pool", time.time() - t0)
            p = np.random.default_rng(2).integers(0, 10000, n)
            x = r[p]
            sg = sig[p]
            proj = np.einsum("kd,ksd->ks", u, pts[sg])
            g = sg[np.arange(n), np.argmax(proj, 1)].astype(np.int32)
            run("c2 vertex-start (config 2)", ns, x, u, g[:, None])
    if "c5edge" in which:
        pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
        ns = vb.NodeSet(pts)
        seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
        run("c5 edge rays N=1e6 d=8", ns, *edge_rays(ns, pts, seeds))
    if "c3edge" in which:
        pts = np.random.default_rng(0).standard_normal((10000, 5))
        ns = vb.NodeSet(pts)
        seeds = np.random.default_rng(1).choice(10000, 10000, replace=False)
        run("c3 edge rays N=1e4 d=5", ns, *edge_rays(ns, pts, seeds))
    if "c5gen" in which:
        pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
        ns = vb.NodeSet(pts)
        rng = np.random.default_rng(4)
        n = 200_000
        g = rng.integers(0, 10 ** 6, n).astype(np.int32)
        u = rng.standard_normal((n, 8))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        run("c5 generator-start N=1e6 d=8", ns, pts[g], u, g[:, None],
            modes=("pruned",))
    if "c4mc" in which:
        pts = np.random.default_rng(0).random((100000, 4))
        ns = vb.NodeSet(pts)
        import paper_2405_10050_b200.integrate_mc as im
        for mode, order in (("pruned", False), ("pruned", False), ("pruned", True), ("pruned", True)):
            im.MC_ORDER_RAYS = order
            torch.cuda.synchronize()
            t0 = time.time()
            vb.mc_cells(ns, np.arange(100000), 1000, seed=0, mode=mode)
            torch.cuda.synchronize()
            print(f"c4 MC 1e8 rays {mode} order={order}: {time.time() - t0:.3f} s "
                  f"({1e8 / (time.time() - t0):.3e} rays/s)", flush=True)
