"""Where does the end-to-end (host arrays) time go?  H2D / D2H bandwidth and
HostRaycaster chunk sizes on config-2-shaped rays."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.raycast import HostRaycaster  # noqa: E402

n, d = 1_000_000, 6
pts = np.random.default_rng(0).random((20000, d))
ns = vb.NodeSet(pts)
if len(sys.argv) > 1 and sys.argv[1] == "config2":
    # the bench's config-2 rays (descent-vertex origins)
    import bench
    s, p_all, u_all = bench.ray_recipe(n)
    need = np.unique(p_all)
    sig_n, r_n = vb.descent_batch(ns, s[need], seed=0)
    pool_sig = np.zeros((bench.N_POOL, d + 1), dtype=np.int32)
    pool_r = np.zeros((bench.N_POOL, d))
    pool_sig[need], pool_r[need] = sig_n, r_n
    xv, u, g1 = bench.assemble(pts, pool_sig, pool_r, p_all, u_all)
    g = g1[:, 0]
else:
    rng = np.random.default_rng(3)
    g = rng.integers(0, 20000, n).astype(np.int32)
    u = rng.standard_normal((n, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    xv = pts[g]
P = HostRaycaster.pinned
hx, hu, hg = P((n, d), torch.float64), P((n, d), torch.float64), P((n, 1), torch.int32)
hx.copy_(torch.from_numpy(np.ascontiguousarray(xv)))
hu.copy_(torch.from_numpy(u))
hg.copy_(torch.from_numpy(np.ascontiguousarray(g[:, None], dtype=np.int32)))
dx = torch.empty((n, d), dtype=torch.float64, device="cuda")
for name, src, dst in (("H2D 48MB", hx, dx), ("D2H 48MB", dx, hx)):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {dt * 1e3:.2f} ms = {48e6 / dt / 1e9:.1f} GB/s")
ref_idx = vb.raycast_batch(ns, hx.cuda(), hu.cuda(), hg.cuda()).idx.cpu().numpy()
hidx, ht = P((n,), torch.int32), P((n,), torch.float64)
hrp, hfl = P((n, d), torch.float64), P((n,), torch.uint8)
for chunk, minc, graphs, nb, cst in ((1 << 19, 1 << 19, False, 4, 2), (1 << 18, 1 << 16, True, 4, 2),
                                    (1 << 18, 1 << 16, True, 8, 4), (1 << 17, 1 << 15, True, 8, 4),
                                    (1 << 17, 1 << 16, True, 8, 4), (1 << 17, 1 << 17, True, 8, 4),
                                    (1 << 16, 1 << 16, True, 16, 8), (1 << 18, 1 << 15, True, 8, 4),
                                    (1 << 19, 1 << 15, True, 8, 4), (1 << 19, 1 << 16, True, 4, 4),
                                    (1 << 18, 1 << 14, True, 8, 4), (1 << 18, 1 << 15, True, 8, 8)):
    hr = HostRaycaster(ns, n, 1, chunk=chunk, min_chunk=minc, graphs=graphs, nbuf=nb,
                       compute_streams=cst)
    hr.run(hx, hu, hg, hidx, ht, hrp, hfl)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        hr.run(hx, hu, hg, hidx, ht, hrp, hfl)
    dt = (time.perf_counter() - t0) / 3
    t0 = time.perf_counter()
    hr.run(hx, hu, hg, hidx, ht, hrp, hfl, sync=False)
    te = time.perf_counter() - t0
    torch.cuda.synchronize()
    ok = np.array_equal(hidx.numpy(), ref_idx)
    print(f"graphs={graphs} bufs={nb} streams={cst} chunk {chunk} min {minc}: {dt * 1e3:.2f} ms  {n / dt:.3e} rays/s  (host enqueue {te * 1e3:.2f} ms) same={ok}")
