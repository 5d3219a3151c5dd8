"""Host-side time per traversal level (config 1 / config 3): the native
open / cast calls (each ends with a stream sync) and the rest of the level."""
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200 import _lib  # noqa: E402

acc = defaultdict(float)
cnt = defaultdict(int)
L = _lib.lib()


def wrap(name):
    f = getattr(L, name)

    def g(*a):
        t0 = time.perf_counter()
        r = f(*a)
        acc[name] += time.perf_counter() - t0
        cnt[name] += 1
        return r
    setattr(L, name, g)


for nm in ("vr_trav_level_open", "vr_trav_level_cast", "vr_trav_finalize", "vr_trav_boundary",
           "vr_trav_level_workspace", "vr_trav_edge_compact", "vr_trav_published"):
    wrap(nm)
for name, pts in (("config1", np.random.default_rng(0).random((1000, 3))),
                  ("config3", np.random.default_rng(0).standard_normal((10000, 5)))):
    ns = vb.build_node_set(pts)
    vb.voronoi_graph(ns, seed=0)
    acc.clear(); cnt.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m, info = vb.voronoi_graph(ns, seed=0, return_info=True)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"{name}: total {tot * 1e3:.2f} ms, {len(info['levels'])} levels")
    for k in sorted(acc, key=lambda k: -acc[k]):
        print(f"   {k:28s} {acc[k] * 1e3:8.3f} ms  x{cnt[k]}")
    print(f"   rest (python, descent, tables): {(tot - sum(acc.values())) * 1e3:.3f} ms")
