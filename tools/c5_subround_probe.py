"""Coherence cost of splitting a config-5 level into S sub-rounds: the edge
rays of half the level-4 vertices cast in one launch vs S launches over the
vertices with id % S == j (sum of the S kernel times)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402

dev = torch.device("cuda", 0)
d = 8
pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts)
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
mesh, lv = vb.voronoi_local(ns, seeds, hops=4, return_levels=True)
dv = mesh.device_arrays()
sel = np.nonzero(lv == 4)[0]
sel = np.sort(np.random.default_rng(2).choice(sel, len(sel) // 2, replace=False))
sd = dv["sigma"][torch.as_tensor(sel, device=dev)]
rd = dv["r"][torch.as_tensor(sel, device=dev)]
u, ok = vb.vertex_directions_batch(ns, sd)
nv = sd.shape[0]
keep = torch.ones((d + 1, d + 1), dtype=torch.bool, device=dev) ^ torch.eye(d + 1, dtype=torch.bool, device=dev)
del mesh, dv
torch.cuda.empty_cache()


def rays(vsel):
    s, r, uu, okk = sd[vsel], rd[vsel], u[vsel], ok[vsel]
    m = s.shape[0]
    x = r.repeat_interleave(d + 1, 0)
    uf = uu.reshape(-1, d)
    eta = s[:, None, :].expand(m, d + 1, d + 1)[:, keep].reshape(m * (d + 1), d).contiguous()
    okf = okk.reshape(-1).bool()
    return x[okf].contiguous(), uf[okf].contiguous(), eta[okf].contiguous()


def cast(x, uf, eta):
    ts = []
    for i in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        vb.raycast_batch(ns, x, uf, eta, want_rp=False, events=ev)
        torch.cuda.synchronize()
        if i:
            ts.append(ev[0].elapsed_time(ev[2]))
    return float(np.median(ts)), x.shape[0]


# split by direction instead: sign of the dominant component (2 rounds),
# dominant axis parity x sign (4 rounds)
X, U, E = rays(torch.arange(nv, device=dev))
dom = U.abs().argmax(1)
sgn = (U.gather(1, dom[:, None])[:, 0] > 0).long()
for name, cls, S in (("sign", sgn, 2), ("axis-parity x sign", (dom % 2) * 2 + sgn, 4),
                     ("axis", dom, 8)):
    tot = 0.0
    for j in range(S):
        m = cls == j
        t, _ = cast(X[m].contiguous(), U[m].contiguous(), E[m].contiguous())
        tot += t
    print(f"direction split {name} S={S}: total {tot:.1f} ms", flush=True)
del X, U, E
ids = torch.arange(nv, device=dev)
for S in (1, 2, 4, 8):
    tot = 0.0
    n = 0
    for j in range(S):
        t, m = cast(*rays(ids[ids % S == j]))
        tot += t
        n += m
    print(f"S={S}: rays {n} total {tot:.1f} ms ({tot / n * 1e3:.3f} us/ray)", flush=True)
