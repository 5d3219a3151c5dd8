"""CPU oracle for the incircle RayCast hot path -- TEST INFRASTRUCTURE ONLY.

This module is a restatement of the reference algorithm (arXiv 2405.10050's
`voronray`, pkg/src/voronray/*.py) in numpy + scipy.  It exists to CHECK the
B200 product path and to time the reference's CPU algorithm on the GPU box's
host cores.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
/ reference legs may import it; the product package never does (there is no
CPU fallback in paper_2405_10050_b200).

Pinning: tests/test_oracle.py checks this restatement against golden vectors
produced by running the unmodified reference in the build container
(tests/golden/make_golden.py, make_golden_heavy.py) -- raycast indices and
coordinates, descent vertices, full-diagram sigma sets and digests, and MC
areas/volumes under replayed normals.

Third-party dependency on the path: scipy.spatial.cKDTree (not vendored by
the reference; `scipy>=1.10` unpinned, pkg/pyproject.toml:10-14).  It is the
same library here (scipy 1.18.1), used exactly where the reference uses it:
the NN probe for N > 2048 (core.py:52-57, 92-103).
"""

from __future__ import annotations

import hashlib
import math

import numpy as np
from scipy.spatial import cKDTree

TOL_VERTEX = 1e-8          # core.py:24
TOL_DEGENERATE = 1e-10     # core.py:27
HALFSPACE_SLACK = 1e-12    # core.py:29
SCAN_MAX = 2048            # core.py:32
DESCENT_RETRIES = 100      # graph.py:25
RANK_TOL = 1e-10           # raycast.py:28
PURPOSES = {"descent": 0, "mc": 1, "bench": 2, "test": 3}  # rng.py:10-15


class Degenerate(Exception):
    """Restates DegenerateConfiguration (errors.py:16)."""


class Escaped(Exception):
    """Restates UnboundedRay (errors.py:32-38)."""

    def __init__(self, cell, direction):
        super().__init__(cell)
        self.cell, self.direction = cell, direction


class Retry(Exception):
    """Restates RetryExhausted (errors.py:28)."""


def stream(seed, purpose, index=0):
    """rng.py:18-28: SeedSequence(entropy=seed, spawn_key=(tag, index)) -> PCG64."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(PURPOSES[purpose], index))
    return np.random.Generator(np.random.PCG64(ss))


class Nodes:
    """Generator set with the reference's two NN backends (core.py:35-142)."""

    def __init__(self, points, backend="auto"):
        self.p = np.ascontiguousarray(np.array(points, dtype=float))
        self.n, self.d = self.p.shape
        self.sq = np.einsum("ij,ij->i", self.p, self.p)
        if backend == "auto":
            backend = "scan" if self.n <= SCAN_MAX else "kdtree"
        self.backend = backend
        self.tree = cKDTree(self.p) if backend == "kdtree" else None

    def tree_nearest(self, q, skip, want_second=False):
        """Expanding-k kd-tree query with a skip predicate (core.py:92-103,
        113-128)."""
        k = 8 if want_second else 4
        while True:
            kk = min(k, self.n)
            dist, idx = self.tree.query(q, k=kk)
            found = []
            for dd, ii in zip(np.atleast_1d(dist), np.atleast_1d(idx)):
                if ii < self.n and not skip(int(ii)):
                    found.append((int(ii), float(dd)))
                    if not want_second or len(found) == 2:
                        return found if want_second else found[0]
            if kk == self.n:
                if not found:
                    return None
                return found + [(None, math.inf)] if want_second else found[0]
            k *= 4


class Probe:
    """Forward-halfspace NN probe of one raycast (raycast.py:85-151)."""

    def __init__(self, nodes, eta, u, candidates=None):
        p = nodes.p
        thr = float(np.max(p[list(eta)] @ u)) if len(eta) > 1 else float(p[eta[0]] @ u)
        self.thr = thr + HALFSPACE_SLACK * max(1.0, abs(thr))
        self.nodes, self.u = nodes, u
        if candidates is not None:
            self.idx = np.asarray(candidates, dtype=np.intp)
            self.cp = p[self.idx]
            csq = np.einsum("ij,ij->i", self.cp, self.cp)
        elif nodes.tree is None:
            self.idx, self.cp, csq = None, p, nodes.sq
        else:
            self.idx, self.cp = None, None
            return
        bad = (self.cp @ u) <= self.thr
        self.none_valid = bool(bad.all())
        self.csq = np.where(bad, np.inf, csq)

    def __call__(self, q):
        if self.cp is not None:
            if self.none_valid:
                return None
            self.d2 = self.csq - 2.0 * (self.cp @ q)
            k = int(np.argmin(self.d2))
            self.qq = float(q @ q)
            i = int(self.idx[k]) if self.idx is not None else k
            return i, math.sqrt(max(self.d2[k] + self.qq, 0.0))
        p, u, thr = self.nodes.p, self.u, self.thr
        self.q = q
        return self.nodes.tree_nearest(q, lambda i: float(p[i] @ u) <= thr)

    def second(self):
        if self.cp is not None:
            if len(self.d2) < 2:
                return math.inf
            return math.sqrt(max(float(np.partition(self.d2, 1)[1]) + self.qq, 0.0))
        p, u, thr = self.nodes.p, self.u, self.thr
        res = self.nodes.tree_nearest(self.q, lambda i: float(p[i] @ u) <= thr, want_second=True)
        return math.inf if res is None else res[1][1]


def raycast(nodes, eta, r, u, candidates=None, heuristic=False, counter=None):
    """The incircle probe loop (raycast.py:154-224).

    Returns (sorted sigma, rp), None on escape; raises Degenerate."""
    p = nodes.p
    x0 = p[eta[0]]
    probe = Probe(nodes, eta, u, candidates)
    anchor = r
    if heuristic and len(eta) == nodes.d:
        # regular-simplex warm start (raycast.py:68-82): result-neutral
        rp0 = r + u * float(u @ (x0 - r))
        rad = math.sqrt(float((rp0 - x0) @ (rp0 - x0)))
        anchor = rp0 + u * (rad / math.sqrt((len(eta) - 1) * (len(eta) + 1)))
    hit = probe(anchor)
    if counter is not None:
        counter[0] += 1
    if hit is None:
        return None
    i = hit[0]
    b = r - x0
    base, b_u, ux0 = float(b @ b), float(u @ b), float(u @ x0)
    prev = math.inf
    while True:
        a = r - p[i]
        t = (float(a @ a) - base) / (2.0 * (float(u @ p[i]) - ux0))
        if not t < prev:
            raise Degenerate("stall")
        prev = t
        rp = r + t * u
        radius = math.sqrt(max(base + t * (2.0 * b_u + t), 0.0))
        j, dj = probe(rp)
        if counter is not None:
            counter[0] += 1
        if j == i:
            if probe.second() < radius * (1.0 + TOL_DEGENERATE):
                raise Degenerate("runner-up on the circumsphere")
            return tuple(sorted((*eta, i))), rp
        if dj >= radius * (1.0 - TOL_DEGENERATE):
            raise Degenerate("probe hit on the circumsphere")
        i = j


def raycast_argmin(points, x, u, eta, sq=None):
    """Vectorised closed form of the same answer: argmin over
    valid i of t_i, smallest index on ties; -1 when nothing is valid.
    x, u: (n, d); eta: (n, k).  Returns (idx, t) with the winner's t from the
    reference's centred formula."""
    p = np.asarray(points, dtype=float)
    x = np.atleast_2d(x)
    u = np.atleast_2d(u)
    eta = np.atleast_2d(eta)
    n = x.shape[0]
    idx = np.full(n, -1, dtype=np.int64)
    tt = np.full(n, np.inf)
    for k in range(n):
        uu, xx = u[k], x[k]
        thr = float(np.max(p[eta[k]] @ uu))
        thr += HALFSPACE_SLACK * max(1.0, abs(thr))
        q = p @ uu
        valid = q > thr
        if not valid.any():
            continue
        xg = p[eta[k][0]]
        base = float((xx - xg) @ (xx - xg))
        diff = p[valid] - xx
        num = np.einsum("ij,ij->i", diff, diff) - base
        t = num / (2.0 * (q[valid] - float(uu @ xg)))
        w = int(np.argmin(t))
        i = int(np.nonzero(valid)[0][w])
        a = xx - p[i]
        idx[k] = i
        tt[k] = (float(a @ a) - base) / (2.0 * (float(uu @ p[i]) - float(uu @ xg)))
    return idx, tt


def orthonormal_rows(diffs):
    """Two-pass modified Gram-Schmidt (raycast.py:295-308)."""
    out = []
    for row in diffs:
        v = np.array(row, dtype=float)
        n0 = math.sqrt(float(v @ v))
        for _ in range(2):
            for q in out:
                v -= (q @ v) * q
        nv = math.sqrt(float(v @ v))
        if nv < RANK_TOL * max(n0, 1.0):
            raise Degenerate("affinely dependent")
        out.append(v / nv)
    return out


def project_out(w, basis):
    v = np.array(w, dtype=float)
    for _ in range(2):
        for q in basis:
            v -= (q @ v) * q
    return v


def vertex_directions(p, sigma, positions):
    """Columns of D^-1 (raycast.py:345-378)."""
    sub = p[list(sigma)]
    inv = np.linalg.inv(sub[1:] - sub[0])
    out = {}
    for k in positions:
        v = inv.sum(axis=1) if k == 0 else -inv[:, k - 1]
        out[k] = v / math.sqrt(float(v @ v))
    return out


def descent(nodes, start, rng, counter=None):
    """graph.py:46-85 (incircle raycaster; the heuristic is result-neutral)."""
    p, d = nodes.p, nodes.d
    sigma, r = (int(start),), np.array(p[start], dtype=float)
    fails, basis = 0, []
    while len(sigma) < d + 1:
        u = project_out(rng.standard_normal(d), basis)
        nrm = np.linalg.norm(u)
        if nrm < 1e-9:
            continue
        res = raycast(nodes, sigma, r, u / nrm, counter=counter)
        if res is None:
            fails += 1
            if fails >= DESCENT_RETRIES:
                raise Retry(start)
            continue
        sigma, r = res
        fails = 0
        basis = orthonormal_rows(p[list(sigma[1:])] - p[sigma[0]])
    return sigma, r


def voronoi_graph(nodes, seed=0, counter=None):
    """Depth-first edge-counting traversal (graph.py:88-146).

    Returns (vertices: dict sigma -> r, edge_counts: dict, boundary: list of
    (sigma, u), raycasts)."""
    p = nodes.p
    verts, counts, boundary, stack = {}, {}, [], []
    nray = [0]

    def discover(s, r):
        verts[s] = r
        for k in range(len(s)):
            e = s[:k] + s[k + 1:]
            counts[e] = counts.get(e, 0) + 1
        stack.append((s, r))

    s0, r0 = descent(nodes, 0, stream(seed, "descent", 0), counter=counter)
    discover(s0, r0)
    while stack:
        s, r = stack.pop()
        open_ks = [k for k in range(len(s)) if counts.get(s[:k] + s[k + 1:], 0) < 2]
        if not open_ks:
            continue
        dirs = vertex_directions(p, s, open_ks)
        for k in open_ks:
            eta = s[:k] + s[k + 1:]
            if counts.get(eta, 0) >= 2:
                continue
            nray[0] += 1
            res = raycast(nodes, eta, r, dirs[k], heuristic=True, counter=counter)
            if res is None:
                boundary.append((s, dirs[k]))
            elif res[0] not in verts:
                discover(*res)
    return verts, counts, boundary, nray[0]


def unit(y):
    return y / math.sqrt(float(y @ y))


def mc_areas(nodes, i, n, rng, neighbors=None):
    """mc_areas_only (integrate_mc.py:124-161) and its neighbour batch form
    (integrate_mc.py:164-197).  Returns (areas, volume, samples)."""
    p, d = nodes.p, nodes.d
    xi = p[i]
    surf = 2.0 * math.pi ** (d / 2.0) / math.gamma(d / 2.0)
    if neighbors is not None and len(neighbors) > 0:
        nb = np.asarray(neighbors, dtype=np.intp)
        diffs = p[nb] - xi
        dist2 = np.einsum("kd,kd->k", diffs, diffs)
        y = rng.standard_normal((n, d))
        y /= np.linalg.norm(y, axis=1, keepdims=True)
        den = 2.0 * (y @ diffs.T)
        with np.errstate(divide="ignore", invalid="ignore"):
            t = np.where(den > 0.0, dist2[None, :] / den, np.inf)
        k = np.argmin(t, axis=1)
        rows = np.arange(n)
        length = t[rows, k]
        bad = ~np.isfinite(length)
        if bad.any():
            raise Escaped(i, y[int(np.nonzero(bad)[0][0])])
        cos = 0.5 * den[rows, k] / np.sqrt(dist2[k])
        acc = np.zeros(len(nb))
        np.add.at(acc, k, length ** (d - 1) / cos)
        samples = length ** d
        return ({int(j): float(a) * surf / n for j, a in zip(nb, acc) if a > 0.0},
                float(samples.sum()) * surf / (d * n), samples)
    area, vol = {}, 0.0
    samples = np.empty(n)
    for k in range(n):
        while True:
            z = rng.standard_normal(d)
            if math.sqrt(float(z @ z)) > 0.0:
                y = unit(z)
                break
        res = raycast(nodes, (i,), xi, y)
        if res is None:
            raise Escaped(i, y)
        sig, rp = res
        j = sig[1] if sig[0] == i else sig[0]
        seg = rp - xi
        length = math.sqrt(float(seg @ seg))
        nij = p[j] - xi
        cos = float(nij @ y) / math.sqrt(float(nij @ nij))
        area[j] = area.get(j, 0.0) + length ** (d - 1) / cos
        samples[k] = length ** d
        vol += length ** d
    return ({j: a * (surf / n) for j, a in area.items()}, vol * surf / (d * n), samples)


def circumcenter(p, sigma):
    """fp64 solve of 2(x_s - x_s0).y = |x_s - x_s0|^2, r = x_s0 + y (the
    coordinate reference of SURVEY.md §8(c) rule 3, centred form)."""
    sub = p[list(sigma)]
    dd = sub[1:] - sub[0]
    return sub[0] + np.linalg.solve(2.0 * dd, np.einsum("ij,ij->i", dd, dd))


def verify_vertex(p, sigma, r, tol=TOL_VERTEX):
    """core.py:279-296."""
    sig = list(sigma)
    dists = np.linalg.norm(p[sig] - r, axis=1)
    rad = dists[0]
    if rad <= 0.0 or np.max(np.abs(dists - rad)) > tol * rad:
        return False
    d2 = np.linalg.norm(p - r, axis=1)
    d2[sig] = np.inf
    return bool(np.min(d2) >= rad * (1.0 - tol))


def sigma_digest(sigmas):
    """sha256 of the sorted sigma array as little-endian int32."""
    arr = np.asarray(sorted(tuple(int(x) for x in s) for s in sigmas), dtype="<i4")
    return hashlib.sha256(arr.tobytes()).hexdigest()


# --- Philox4x32-10 + Box-Muller: numpy port of the device direction stream ---
_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def _philox(c0, c1, c2, c3, k0, k1):
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint32) for v in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    for _ in range(10):
        p0 = c0.astype(np.uint64) * _M0
        p1 = c2.astype(np.uint64) * _M1
        hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & _MASK).astype(np.uint32)
        hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & _MASK).astype(np.uint32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = np.uint32((int(k0) + int(_W0)) & 0xFFFFFFFF)
        k1 = np.uint32((int(k1) + int(_W1)) & 0xFFFFFFFF)
    return c0, c1, c2, c3


def philox_normals(seed, cells, n, d):
    """Raw Gaussian draws of the device MC stream for cells x n rays, shape
    (len(cells)*n, d); matches csrc/raycast_core.cuh philox_normals up to the
    last-ulp differences of log / sincos between libm and CUDA."""
    cells = np.asarray(cells, dtype=np.int64)
    ray = np.tile(np.arange(n, dtype=np.int64), len(cells))
    cell = np.repeat(cells, n)
    out = np.empty((len(ray), d))
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    for pi in range((d + 1) // 2):
        c0 = (ray & 0xFFFFFFFF).astype(np.uint32)
        c1 = (cell & 0xFFFFFFFF).astype(np.uint32)
        c2 = (np.uint32(pi) | ((ray >> 32).astype(np.uint32) << np.uint32(8))).astype(np.uint32)
        c3 = (np.uint32(0x4D430000) | ((cell >> 32) & 0xFFFF).astype(np.uint32)).astype(np.uint32)
        w0, w1, w2, w3 = _philox(c0, c1, c2, c3, seed & 0xFFFFFFFF, seed >> 32)
        a = ((w0.astype(np.uint64) << np.uint64(32)) | w1.astype(np.uint64)) >> np.uint64(11)
        b = ((w2.astype(np.uint64) << np.uint64(32)) | w3.astype(np.uint64)) >> np.uint64(11)
        u1 = (a + np.uint64(1)).astype(np.float64) * 2.0 ** -53
        u2 = b.astype(np.float64) * 2.0 ** -53
        rad = np.sqrt(-2.0 * np.log(u1))
        ang = 6.283185307179586 * u2
        out[:, 2 * pi] = rad * np.cos(ang)
        if 2 * pi + 1 < d:
            out[:, 2 * pi + 1] = rad * np.sin(ang)
    return out


class Replay:
    """Duck-typed rng serving pre-drawn normals in order."""

    def __init__(self, z):
        self.z = np.asarray(z, dtype=float).ravel()
        self.pos = 0

    def standard_normal(self, size=None):
        m = 1 if size is None else int(np.prod(size))
        out = self.z[self.pos:self.pos + m]
        self.pos += m
        return float(out[0]) if size is None else out.reshape(size).copy()
