"""Full-diagram traversal timing (configs 1 and 3) with per-level detail."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
import paper_2405_10050_b200.raycast as _rc  # noqa: E402

if os.environ.get("PRUNE_MIN"):
    _rc.PRUNE_MIN_GENERATORS = int(os.environ["PRUNE_MIN"])

for name, pts in (("config1", np.random.default_rng(0).random((1000, 3))),
                  ("config3", np.random.default_rng(0).standard_normal((10000, 5)))):
    ns = vb.build_node_set(pts)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = vb.RaycastStats()
        mesh, info = vb.voronoi_graph(ns, seed=0, stats=st, return_info=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{name} rep{rep}: {dt:.3f} s  V={info['vertices']} B={info['boundary']} "
              f"levels={len(info['levels'])} raycasts={st.raycasts} "
              f"-> {info['vertices'] / dt:.3e} vertices/s", flush=True)
    print("  max frontier", max(f for f, _ in info["levels"]))
