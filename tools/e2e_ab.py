"""Config-2 e2e (HostRaycaster.run, pinned host arrays) and device times for
the whole 1e6-ray batch and for sparse slices, under the loaded library
(VR_LIB_PATH selects a variant build)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.raycast import HostRaycaster  # noqa: E402

pts = bench.generators()
ns = vb.build_node_set(pts)
n = 10 ** 6
s, p, uu = bench.ray_recipe(n)
need = np.unique(p)
sig, r = vb.descent_batch(ns, s[need], seed=0)
ps = np.zeros((bench.N_POOL, 7), dtype=np.int32)
pr = np.zeros((bench.N_POOL, 6))
ps[need], pr[need] = sig, r
x, u, g = bench.assemble(pts, ps, pr, p, uu)
xd, ud, gd = (torch.from_numpy(t).cuda() for t in (x, u, g))


def dev_ms(lo, hi, reps=5):
    ts = []
    for i in range(reps + 2):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        vb.raycast_batch(ns, xd[lo:hi], ud[lo:hi], gd[lo:hi], events=ev)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(ev[0].elapsed_time(ev[2]))
    return float(np.median(ts))


full = dev_ms(0, n)
s256 = dev_ms(0, 1 << 18)
s64 = dev_ms(0, 1 << 16)
kw = {}
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    kw[k] = int(v)
hr = HostRaycaster(ns, n, 1, **kw)
pin = HostRaycaster.pinned
hx, hu, hg = pin(x.shape, torch.float64), pin(u.shape, torch.float64), pin(g.shape, torch.int32)
hx.copy_(torch.from_numpy(x)); hu.copy_(torch.from_numpy(u)); hg.copy_(torch.from_numpy(g))
hidx, ht = pin((n,), torch.int32), pin((n,), torch.float64)
hrp, hfl = pin((n, 6), torch.float64), pin((n,), torch.uint8)
for _ in range(3):
    hr.run(hx, hu, hg, hidx, ht, hrp, hfl)
ts = []
for _ in range(7):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hr.run(hx, hu, hg, hidx, ht, hrp, hfl)
    ts.append((time.perf_counter() - t0) * 1e3)
e2e = float(np.median(ts))
# pure copies of the same bytes (pinned, one stream each direction)
dx = torch.empty_like(xd); du = torch.empty_like(ud); dg = torch.empty_like(gd)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record(); dx.copy_(hx, non_blocking=True); du.copy_(hu, non_blocking=True)
dg.copy_(hg, non_blocking=True); ev[1].record()
hrp.copy_(torch.empty((n, 6), dtype=torch.float64, device="cuda"), non_blocking=True); ev[2].record()
torch.cuda.synchronize()
print(f"{os.environ.get('VR_LIB_PATH', 'base')} {kw}: device full {full:.3f} ms per 1e6; "
      f"256k slice {s256 * n / (1 << 18):.3f} ms per 1e6; 64k slice {s64 * n / (1 << 16):.3f} ms per 1e6; "
      f"e2e {e2e:.3f} ms = {n / e2e / 1e3:.1f} M rays/s; H2D 100 MB {ev[0].elapsed_time(ev[1]):.3f} ms, "
      f"D2H 48 MB {ev[1].elapsed_time(ev[2]):.3f} ms")
