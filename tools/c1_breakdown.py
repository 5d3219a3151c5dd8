"""Config-1 (N=1000, d=3) full-diagram time by phase: descent, table setup,
the native level loop, edge extraction, Mesh construction (ms, median of 5)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200 import graph as G  # noqa: E402
from paper_2405_10050_b200 import rng as _rng  # noqa: E402
from paper_2405_10050_b200.raycast import Workspace  # noqa: E402

pts = np.random.default_rng(0).random((1000, 3))
ns = vb.build_node_set(pts)
vb.voronoi_graph(ns, seed=0)
rows = []
for rep in range(6):
    T = {}

    def mark(k, t0):
        torch.cuda.synchronize()
        T[k] = (time.perf_counter() - t0) * 1e3
        return time.perf_counter()
    torch.cuda.synchronize()
    t = t0 = time.perf_counter()
    st = vb.RaycastStats()
    first = G.descent(ns, 0, _rng.stream(0, "descent", 0), st)
    t = mark("descent", t)
    v_est = G._table_estimate(ns, ns.n * 7)
    tr = G.DeviceTraversal(ns, vcap_hint=max(4 * ns.n, 2 * v_est), ecap_hint=2 * 4 * v_est)
    tr.seed_vertex(first.sigma)
    ws = Workspace()
    t = mark("tables", t)
    news, _, _ = tr.run(0, 1, 1, -1, stats=st, ws=ws)
    t = mark("levels", t)
    ek, ec = tr.edges()
    t = mark("edges", t)
    mesh = vb.Mesh.from_device(ns, tr.vsig[:tr.nv], tr.vr[:tr.nv], ek, ec, tr.bsig[:tr.nb],
                               tr.bu[:tr.nb])
    t = mark("mesh", t)
    T["total"] = (t - t0) * 1e3
    T["levels_n"] = len(news)
    rows.append(T)
for k in rows[0]:
    print(f"{k:10s} {np.median([r[k] for r in rows[1:]]):8.3f}")
ts = []
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vb.voronoi_graph(ns, seed=0)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("voronoi_graph median ms", np.median(ts[1:]))
