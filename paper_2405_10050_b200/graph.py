"""Vertex descent and the exhaustive traversal on the B200.

Drop-in for pkg/src/voronray/graph.py.

* ``descent`` keeps the reference algorithm and RNG consumption exactly
  (graph.py:46-85): directions come from the caller's host stream, each level
  is one GPU RayCast.  ``descent_batch`` runs many descents at once, one GPU
  launch per level group.
* ``voronoi_graph`` replaces the depth-first stack (graph.py:88-146) with a
  level-synchronous frontier traversal on the device (csrc/traverse.cu):
  open-edge test against a device edge-count table, batched edge directions,
  the fused RayCast over all open edges of the level, deterministic
  claim-and-dedupe of the new sigma keys in a device hash set, fresh fp64
  circumcentres for new vertices, and edge-count bumps.  The vertex set, the
  edge counts and the boundary-ray multiset equal the reference's; vertex
  coordinates are the fp64 circumcentre of sigma (SURVEY.md §8(c) rule 3).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from itertools import combinations

import numpy as np
import torch

from . import _lib
from . import rng as _rng
from .core import (TOL_VERTEX, Mesh, NodeSet, VertexRecord, edge_keys, verify_vertices)
from .errors import RetryExhausted
from .raycast import (RayQuery, RaycastStats, _orthonormal_rows, _project_out, raycast_batch,
                      raycast_incircle)

DESCENT_RETRIES = 100


def edge_set(sigma):
    """The d+1 edges of a vertex (graph.py:28-31)."""
    sigma = tuple(sigma)
    return set(edge_keys(sigma))


def _resolve_raycaster(method, eps):
    if method in ("incircle_heuristic", "incircle"):
        return lambda ns, q, stats: raycast_incircle(ns, q, stats)
    if method == "bisection":
        raise ValueError("the bisection baseline (raycast.py:227-292) is a CPU benchmark "
                         "baseline and is not part of the B200 build")
    raise ValueError(f"unknown raycast method {method!r}")


def descent(ns: NodeSet, start_index: int, rng=None, stats: RaycastStats = None,
            raycaster=None) -> VertexRecord:
    """Find one Voronoi vertex by raycasting onto lower faces (graph.py:46-85).

    Raises:
        RetryExhausted: after 100 consecutive escaped rays at one level.
    """
    if rng is None:
        rng = _rng.stream(0, "descent", start_index)
    if stats is None:
        stats = RaycastStats()
    if raycaster is None:
        raycaster = _resolve_raycaster("incircle_heuristic", None)
    pts = ns.points
    d = ns.dim
    sigma = (int(start_index),)
    r = np.array(pts[start_index], dtype=float)
    failures = 0
    basis = []
    while len(sigma) < d + 1:
        u = rng.standard_normal(d)
        u = _project_out(u, basis)
        norm = np.linalg.norm(u)
        if norm < 1e-9:
            continue  # draw fell into the generator span; free redraw
        res = raycaster(ns, RayQuery(sigma, r, u / norm), stats)
        if res is None:
            failures += 1
            if failures >= DESCENT_RETRIES:
                raise RetryExhausted(f"descent from node {start_index} stuck at level {len(sigma)}")
            continue
        sigma, r = res
        failures = 0
        basis = _orthonormal_rows(pts[list(sigma[1:])] - pts[sigma[0]])
    return VertexRecord(sigma, r)


def descent_batch(ns: NodeSet, starts, seed: int = 0, stats: RaycastStats = None,
                  rngs=None):
    """Many descents at once; same RNG streams and results as calling
    :func:`descent` with ``stream(seed, "descent", s)`` for every start.

    Returns (sigma (S, d+1) int32, r (S, d) fp64)."""
    pts = ns.points
    d = ns.dim
    starts = [int(s) for s in starts]
    S = len(starts)
    if rngs is None:
        rngs = [_rng.stream(seed, "descent", s) for s in starts]
    sig = [(s,) for s in starts]
    rr = [np.array(pts[s], dtype=float) for s in starts]
    basis = [[] for _ in starts]
    fails = [0] * S
    active = list(range(S))
    while active:
        groups = {}
        for a in active:
            while True:
                u = _project_out(rngs[a].standard_normal(d), basis[a])
                norm = np.linalg.norm(u)
                if norm >= 1e-9:
                    break
            groups.setdefault(len(sig[a]), []).append((a, u / norm))
        still = []
        for k, items in sorted(groups.items()):
            ids = [a for a, _ in items]
            x = np.stack([rr[a] for a in ids])
            u = np.stack([v for _, v in items])
            eta = np.array([sig[a] for a in ids], dtype=np.int32).reshape(len(ids), k)
            res = raycast_batch(ns, x, u, eta, stats=stats)
            idx, _, rp, flag = res.to_host()
            for m, a in enumerate(ids):
                if flag[m] == 1:
                    fails[a] += 1
                    if fails[a] >= DESCENT_RETRIES:
                        raise RetryExhausted(
                            f"descent from node {starts[a]} stuck at level {len(sig[a])}")
                    still.append(a)
                    continue
                if flag[m] == 3:
                    from .errors import DegenerateConfiguration
                    raise DegenerateConfiguration(
                        f"degenerate raycast during descent from node {starts[a]}")
                sig[a] = tuple(sorted((*sig[a], int(idx[m]))))
                rr[a] = rp[m]
                fails[a] = 0
                if len(sig[a]) < d + 1:
                    basis[a] = _orthonormal_rows(pts[list(sig[a][1:])] - pts[sig[a][0]])
                    still.append(a)
        active = sorted(still)
    return np.array(sig, dtype=np.int32), np.array(rr, dtype=np.float64)


# ---------------------------------------------------------------------------
# oracles / verification (graph.py:149-245), evaluated on the GPU
# ---------------------------------------------------------------------------

def circumcenters(ns: NodeSet, sigma):
    """fp64 circumcentres of generator tuples (device LU); NaN rows if singular."""
    rec, _ = ns.device_records()
    dev = rec.device
    L = _lib.lib()
    sd = torch.as_tensor(np.ascontiguousarray(sigma, dtype=np.int32), device=dev).view(-1, ns.dim + 1)
    nv = sd.shape[0]
    out = torch.empty((nv, ns.dim), dtype=torch.float64, device=dev)
    ok = torch.empty(nv, dtype=torch.uint8, device=dev)
    _lib.check(L.vr_circumcenters(_lib.ptr(rec), ns.dim, _lib.ptr(sd), nv, _lib.ptr(out),
                                  _lib.ptr(ok), _lib.stream_handle()), "vr_circumcenters")
    return out.cpu().numpy(), ok.cpu().numpy().astype(bool)


def brute_force_vertices(ns: NodeSet, tol: float = TOL_VERTEX, chunk: int = 1 << 18):
    """Subset-enumeration oracle (graph.py:149-180): circumcentres of every
    (d+1)-subset that pass the incircle scan, evaluated on the GPU."""
    n, d = ns.n, ns.dim
    out = {}
    it = combinations(range(n), d + 1)
    while True:
        block = np.array(list(_take(it, chunk)), dtype=np.int32)
        if block.size == 0:
            break
        block = block.reshape(-1, d + 1)
        r, ok = circumcenters(ns, block)
        keep = np.zeros(len(block), dtype=bool)
        if ok.any():
            keep[ok] = verify_vertices(ns, block[ok], r[ok], tol)
        for row in np.nonzero(keep)[0]:
            out[tuple(int(x) for x in block[row])] = r[row].copy()
    return out


def _take(it, k):
    for _, v in zip(range(k), it):
        yield v


@dataclass
class VerifyReport:
    vertices_total: int = 0
    vertex_failures: list = field(default_factory=list)
    edge_failures: list = field(default_factory=list)
    oracle_checked: bool = False
    oracle_missing: list = field(default_factory=list)
    oracle_extra: list = field(default_factory=list)
    oracle_coord_failures: list = field(default_factory=list)

    @property
    def passed(self):
        return not (self.vertex_failures or self.edge_failures or self.oracle_missing or
                    self.oracle_extra or self.oracle_coord_failures)


def verify_mesh(mesh: Mesh, oracle: bool = None, coord_tol: float = 1e-8) -> VerifyReport:
    """Vertex, edge-consistency and (small instances) oracle checks (graph.py:202-245)."""
    ns = mesh.nodes
    verts = mesh.vertices
    report = VerifyReport(vertices_total=len(verts))
    keys = list(verts.keys())
    if keys:
        sig = np.array(keys, dtype=np.int32)
        r = np.array([verts[k].r for k in keys], dtype=np.float64)
        ok = verify_vertices(ns, sig, r)
        report.vertex_failures = [keys[i] for i in np.nonzero(~ok)[0]]
    by_edge = {}
    for s in verts:
        for e in edge_keys(s):
            by_edge.setdefault(e, []).append(s)
    for eta, count in mesh.edge_counts.items():
        incident = by_edge.get(eta, [])
        if count == 2:
            if len(incident) != 2:
                report.edge_failures.append((eta, f"count 2 but {len(incident)} vertices"))
                continue
            if set(incident[0]) & set(incident[1]) != set(eta):
                report.edge_failures.append((eta, "incident sigmas do not intersect in eta"))
        elif count == 1:
            if len(incident) != 1:
                report.edge_failures.append((eta, f"count 1 but {len(incident)} vertices"))
        else:
            report.edge_failures.append((eta, f"invalid count {count}"))
    if oracle is None:
        oracle = ns.dim <= 3 and ns.n <= 200
    if oracle:
        report.oracle_checked = True
        truth = brute_force_vertices(ns)
        ours = {s: v.r for s, v in verts.items()}
        report.oracle_missing = sorted(set(truth) - set(ours))
        report.oracle_extra = sorted(set(ours) - set(truth))
        for s in set(truth) & set(ours):
            if np.linalg.norm(truth[s] - ours[s]) > coord_tol * max(1.0, float(np.linalg.norm(truth[s]))):
                report.oracle_coord_failures.append(s)
    return report


def voronoi_graph(ns, seed=0, *, method="incircle_heuristic", eps=None, stats=None):
    raise NotImplementedError("level-synchronous traversal lands with csrc/traverse.cu")
