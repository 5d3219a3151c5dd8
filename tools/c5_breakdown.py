"""Config-5 (N=1e6, d=8, L=5 around 10k seeds) wall time by phase, as
voronoi_local runs them (ms, median of 3 after a warm pass)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200 import graph as G  # noqa: E402
from paper_2405_10050_b200.raycast import Workspace  # noqa: E402

pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
ns.prune_index()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
rows = []
for rep in range(4):
    T = {}

    def mark(k, t):
        torch.cuda.synchronize()
        T[k] = (time.perf_counter() - t) * 1e3
        return time.perf_counter()
    torch.cuda.synchronize()
    t = t0 = time.perf_counter()
    sig, _ = G.descent_batch(ns, seeds, seed=0)
    _, first = np.unique(sig, axis=0, return_index=True)
    sig = sig[np.sort(first)]
    t = mark("descent", t)
    tr = G.DeviceTraversal(ns, vcap_hint=max(4 * ns.n, 6 * len(sig) * 4 ** 5))
    tr.seed_vertices(sig)
    ws = Workspace()
    t = mark("tables+seed", t)
    news, _, _ = tr.run(0, tr.nv, 1, 5, ws=ws)
    t = mark("levels", t)
    ek, ec = tr.edges()
    t = mark("edges", t)
    mesh = vb.Mesh.from_device(ns, tr.vsig[:tr.nv], tr.vr[:tr.nv], ek, ec, tr.bsig[:tr.nb],
                               tr.bu[:tr.nb])
    t = mark("mesh", t)
    T["total"] = (t - t0) * 1e3
    rows.append(T)
    del mesh, tr, ek, ec
for k in rows[0]:
    print(f"{k:12s} {np.median([r[k] for r in rows[1:]]):9.2f}  {[round(r[k], 1) for r in rows]}")
