"""Rare-path event counts per ray (needs the VR_STATS build, tools/stats_build.sh):
VR_LIB_PATH=paper_2405_10050_b200/build/stats/_voronray_b200.so python tools/rare_stats.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200 import _lib  # noqa: E402

L = _lib.load_library()
L.vr_debug_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
pts = np.random.default_rng(0).random((20000, 6))
ns = vb.NodeSet(pts)
rng = np.random.default_rng(3)
n = 200000
g = rng.integers(0, 20000, n).astype(np.int32)
u = rng.standard_normal((n, 6))
u /= np.linalg.norm(u, axis=1, keepdims=True)
for mode in ("exhaustive", "pruned"):
    for screen in ("fp64", "fp32"):
        vb.raycast_batch(ns, pts[g], u, g[:, None], mode=mode, screen=screen)
        torch.cuda.synchronize()
        L.vr_debug_stats(buf, 1)
        vb.raycast_batch(ns, pts[g], u, g[:, None], mode=mode, screen=screen)
        torch.cuda.synchronize()
        L.vr_debug_stats(buf, 1)
        b = list(buf)
        print(f"{mode:10s} {screen}: blocks/warp-ray {b[0] / (n / 64):8.1f}  rare-blocks frac "
              f"{b[1] / max(b[0], 1):.3f}  entries/ray {b[2] / n:6.2f}  valid/ray {b[3] / n:6.2f}"
              f"  updates/ray {b[4] / n:6.2f}")
