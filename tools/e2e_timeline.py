"""Per-chunk timeline of HostRaycaster.run on the config-2 rays (bench recipe):
when each chunk's H2D copy, RayCast and D2H copy finish (ms from start)."""
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
n = 1_000_000
s, p_all, u_all = bench.ray_recipe(n)
need = np.unique(p_all)
sig_n, r_n = vb.descent_batch(ns, s[need], seed=0)
pool_sig = np.zeros((bench.N_POOL, bench.DIM + 1), dtype=np.int32)
pool_r = np.zeros((bench.N_POOL, bench.DIM))
pool_sig[need], pool_r[need] = sig_n, r_n
x, u, g = bench.assemble(pts, pool_sig, pool_r, p_all, u_all)
P = HostRaycaster.pinned
hx, hu, hg = P(x.shape, torch.float64), P(u.shape, torch.float64), P(g.shape, torch.int32)
hx.copy_(torch.from_numpy(x))
hu.copy_(torch.from_numpy(u))
hg.copy_(torch.from_numpy(g))
hidx, ht = P((n,), torch.int32), P((n,), torch.float64)
hrp, hfl = P((n, bench.DIM), torch.float64), P((n,), torch.uint8)
cfgs = [dict(), dict(chunk=1 << 18, min_chunk=1 << 16), dict(chunk=1 << 19, min_chunk=1 << 16),
        dict(chunk=1 << 19, min_chunk=1 << 17), dict(chunk=3 << 17, min_chunk=1 << 16),
        dict(chunk=1 << 18, min_chunk=1 << 15)]
for cfg in cfgs:
    hr = HostRaycaster(ns, n, 1, **cfg)
    for _ in range(2):
        hr.run(hx, hu, hg, hidx, ht, hrp, hfl)
    torch.cuda.synchronize()
    tr = []
    t0 = time.perf_counter()
    hr.run(hx, hu, hg, hidx, ht, hrp, hfl, trace=tr)
    wall = (time.perf_counter() - t0) * 1e3
    e0 = tr[0]
    print(f"{cfg}: wall {wall:.2f} ms")
    for m, a, b, c in tr[1:]:
        print(f"   chunk {m:7d}: h2d {e0.elapsed_time(a):6.2f}  compute {e0.elapsed_time(b):6.2f}"
              f"  d2h {e0.elapsed_time(c):6.2f}")
dx = torch.from_numpy(x).cuda()
du = torch.from_numpy(u).cuda()
dg = torch.from_numpy(g).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
vb.raycast_batch(ns, dx, du, dg)
torch.cuda.synchronize()
vb.raycast_batch(ns, dx, du, dg, events=ev)
torch.cuda.synchronize()
print(f"device-resident step: {ev[0].elapsed_time(ev[2]):.2f} ms")
for m in (1_000_000, 500_000, 250_000, 131072, 65536):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    vb.raycast_batch(ns, dx[:m], du[:m], dg[:m])
    torch.cuda.synchronize()
    vb.raycast_batch(ns, dx[:m], du[:m], dg[:m], events=ev)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[2])
    print(f"device-resident slice {m:8d}: {ms:.3f} ms  -> {ms * 1e6 / m:.2f} ms per 1e6 rays")
# raw copy-engine rates: 100 MB pinned H2D, 61 MB D2H, alone and concurrent
hb = P((100_000_000,), torch.uint8)
db = torch.empty(100_000_000, dtype=torch.uint8, device="cuda")
hb2 = P((61_000_000,), torch.uint8)
db2 = torch.empty(61_000_000, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        e[0].record(s1); db.copy_(hb, non_blocking=True); e[1].record(s1)
    torch.cuda.synchronize()
    with torch.cuda.stream(s2):
        e[2].record(s2); hb2.copy_(db2, non_blocking=True); e[3].record(s2)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        e[4].record(s1); db.copy_(hb, non_blocking=True)
    with torch.cuda.stream(s2):
        s2.wait_event(e[4]); hb2.copy_(db2, non_blocking=True)
    s1.wait_stream(s2)
    with torch.cuda.stream(s1):
        e[5].record(s1)
    torch.cuda.synchronize()
    print(f"H2D 100 MB {e[0].elapsed_time(e[1]):.3f} ms ({100 / e[0].elapsed_time(e[1]):.1f} GB/s), "
          f"D2H 61 MB {e[2].elapsed_time(e[3]):.3f} ms ({61 / e[2].elapsed_time(e[3]):.1f} GB/s), "
          f"both concurrent {e[4].elapsed_time(e[5]):.3f} ms")
