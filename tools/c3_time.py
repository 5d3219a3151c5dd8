"""Config-3 full diagram (N=10,000, d=5 Gaussian): timed passes with the
library / environment in effect (VR_SUB_RAYS, VR_SUB_MAX, VR_LIB_PATH)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

pts = np.random.default_rng(0).standard_normal((10000, 5))
ns = vb.build_node_set(pts)
ns.prune_index()
ts = []
for rep in range(6):
    st = vb.RaycastStats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mesh, info = vb.voronoi_graph(ns, seed=0, stats=st, return_info=True)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    del mesh
print(f"VR_SUB_RAYS={os.environ.get('VR_SUB_RAYS', '-')} VR_SUB_MAX={os.environ.get('VR_SUB_MAX', '-')}: "
      f"vertices {info['vertices']} raycasts {st.raycasts} levels {len(info['levels'])} "
      f"times {[round(t * 1e3, 1) for t in ts]} ms", flush=True)
