"""Fuzz the tensor-core (tf32) screen's conservativeness: pruned RayCast
(tensor-core screen for d >= 5) vs the exhaustive fp64-screen kernel,
bitwise (index, t, flag), over random distributions, dimensions, scales and
near-degenerate inputs.  usage: python tools/fuzz_screen.py [cases]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402


def points(rng, kind, n, d):
    if kind == "uniform":
        return rng.random((n, d))
    if kind == "gauss":
        return rng.standard_normal((n, d))
    if kind == "cluster":
        c = rng.random((max(2, n // 300), d)) * 50
        return c[rng.integers(0, len(c), n)] + 1e-2 * rng.standard_normal((n, d))
    if kind == "aniso":
        return rng.random((n, d)) * np.exp(rng.uniform(-6, 6, d))
    if kind == "offset":
        return 1e4 + rng.random((n, d)) * 10 ** rng.uniform(-3, 1)
    if kind == "lattice":  # jittered grid: many near-cospherical subsets
        m = int(round(n ** (1.0 / d))) + 1
        g = np.stack(np.meshgrid(*[np.arange(m)] * d, indexing="ij"), -1).reshape(-1, d)[:n]
        return g + 1e-6 * rng.standard_normal(g.shape)
    if kind == "shell":  # points near a sphere: large circumspheres
        v = rng.standard_normal((n, d))
        return v / np.linalg.norm(v, axis=1, keepdims=True) * (1 + 1e-3 * rng.random((n, 1)))
    raise ValueError(kind)


def main(cases):
    rng = np.random.default_rng(12345)
    kinds = ["uniform", "gauss", "cluster", "aniso", "offset", "lattice", "shell"]
    bad = tot = 0
    for c in range(cases):
        d = int(rng.integers(5, 9))
        n = int(rng.integers(2000, 40000))
        kind = kinds[c % len(kinds)]
        pts = points(rng, kind, n, d)
        pts = np.unique(pts, axis=0)
        ns = vb.build_node_set(pts)
        n = len(pts)
        m = 20000
        g = rng.integers(0, n, m)
        u = rng.standard_normal((m, d))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        sets = [(pts[g], u, g[:, None])]
        try:
            sig, r = vb.descent_batch(ns, rng.choice(n, 300, replace=False), seed=c)
            uu, ok = vb.vertex_directions_batch(ns, sig)
            uu = uu.cpu().numpy().reshape(-1, d)
            xs = np.repeat(r, d + 1, axis=0)
            eta = np.array([[s[j] for j in range(d + 1) if j != k] for s in sig
                            for k in range(d + 1)], dtype=np.int32)
            sets.append((xs, uu, eta))
        except Exception as e:  # degenerate descents on lattices are fine to skip
            print(f"case {c} ({kind}, d={d}): descent skipped: {type(e).__name__}")
        for x, uu, eta in sets:
            a = vb.raycast_batch(ns, x, uu, eta, mode="exhaustive", screen="fp64").to_host()
            b = vb.raycast_batch(ns, x, uu, eta, mode="pruned").to_host()
            mis = sum(int((~((p == q) | (np.isnan(p) & np.isnan(q)) if p.dtype.kind == "f"
                             else p == q)).sum()) for p, q in zip(a, b) if p is not None)
            tot += len(x)
            bad += mis
            print(f"case {c:3d} {kind:8s} d={d} n={n:6d} rays={len(x):6d} mismatches={mis}",
                  flush=True)
    print(f"TOTAL rays {tot} mismatching fields {bad}")
    return bad


if __name__ == "__main__":
    sys.exit(1 if main(int(sys.argv[1]) if len(sys.argv) > 1 else 28) else 0)
