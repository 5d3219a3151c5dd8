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

import ctypes
import os

import numpy as np
import torch

from . import _lib
from . import rng as _rng
from .core import (TOL_VERTEX, Mesh, NodeSet, VertexRecord, edge_incidence, edge_keys,
                   verify_vertices, verify_vertices_device)
from .errors import DegenerateConfiguration, RetryExhausted
from .raycast import (PRUNE_MIN_GENERATORS, RANK_TOL, RayQuery, RaycastStats, Workspace,
                      _orthonormal_rows, _project_out, raycast_batch, raycast_incircle)

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


def _mgs_batch(rows):
    """Two-pass modified Gram-Schmidt of each (k, d) row block of `rows`
    (m, k, d), vectorised over m (raycast.py:295-308 per block)."""
    m, k, d = rows.shape
    out = np.zeros_like(rows)
    for j in range(k):
        v = rows[:, j, :].copy()
        n0 = np.sqrt(np.einsum("md,md->m", v, v))
        for _ in range(2):
            for i in range(j):
                qv = out[:, i, :]
                v -= np.einsum("md,md->m", qv, v)[:, None] * qv
        nv = np.sqrt(np.einsum("md,md->m", v, v))
        if np.any(nv < RANK_TOL * np.maximum(n0, 1.0)):
            raise DegenerateConfiguration("generators are affinely dependent")
        out[:, j, :] = v / nv[:, None]
    return out


def _descent_directions(ns, sigma, kcount, z):
    """(v, |v|, bad) for each start: the draw z projected out of the
    Gram-Schmidt basis of its sigma rows (vr_descent_directions)."""
    rec, _ = ns.device_records()
    dev = rec.device
    L = _lib.lib()
    n, d = z.shape
    sd = torch.as_tensor(np.ascontiguousarray(sigma, dtype=np.int32), device=dev)
    kd = torch.as_tensor(np.ascontiguousarray(kcount, dtype=np.int32), device=dev)
    zd = torch.as_tensor(np.ascontiguousarray(z, dtype=np.float64), device=dev)
    v = torch.empty((n, d), dtype=torch.float64, device=dev)
    nrm = torch.empty(n, dtype=torch.float64, device=dev)
    bad = torch.empty(n, dtype=torch.uint8, device=dev)
    _lib.check(L.vr_descent_directions(_lib.ptr(rec), d, _lib.ptr(sd), _lib.ptr(kd), _lib.ptr(zd),
                                       n, RANK_TOL, _lib.ptr(v), _lib.ptr(nrm), _lib.ptr(bad),
                                       _lib.stream_handle()), "vr_descent_directions")
    return v.cpu().numpy(), nrm.cpu().numpy(), bad.cpu().numpy().astype(bool)


def _project_out_batch(w, basis):
    """Component of each w (m, d) orthogonal to its basis rows (m, k, d)."""
    v = w.copy()
    for _ in range(2):
        for i in range(basis.shape[1]):
            qv = basis[:, i, :]
            v -= np.einsum("md,md->m", qv, v)[:, None] * qv
    return v


class _Draws:
    """Standard-normal d-vectors per start, in each start's stream order.

    With the package's own streams (rngs=None) each start's Generator draws
    a block of K vectors at once -- one (K, d) draw equals K sequential (d,)
    draws bitwise -- so the per-level Python loop
    touches no Generator; caller-supplied rngs are drawn from one vector at
    a time so that their state advances exactly as in the reference."""

    def __init__(self, rngs, seed, starts, d, block=None):
        self.d = d
        self.own = rngs is None
        self.rngs = rngs
        if self.own:
            self.K = block or (d + 3)
            S = len(starts)
            self.ptr = np.zeros(S, dtype=np.int64)
            if 0 <= int(seed) < 1 << 64:
                # the package's streams restated over all starts at once in
                # the host library (csrc/host_rng.cu: SeedSequence + PCG64 +
                # NumPy's ziggurat, bit-identical to _rng.stream; ~2 us per
                # start instead of ~20 us for a Generator object)
                self.L = _lib.load_library()
                idx = np.ascontiguousarray(starts, dtype=np.int64)
                self.state = np.zeros((S, 4), dtype=np.uint64)
                _lib.check(self.L.vr_host_streams(int(seed), _rng.PURPOSES["descent"],
                                                  idx.ctypes.data, S, self.state.ctypes.data),
                           "vr_host_streams")
                self.buf = np.empty((S, self.K, d))
                self._draw(None, S, self.buf)
            else:
                self.state = None
                self.rngs = [_rng.stream(seed, "descent", int(s)) for s in starts]
                self.buf = np.stack([g.standard_normal((self.K, d)) for g in self.rngs])

    def _draw(self, rows, n, out):
        _lib.check(self.L.vr_host_normals(self.state.ctypes.data,
                                          None if rows is None else rows.ctypes.data, n,
                                          self.K * self.d, out.ctypes.data), "vr_host_normals")

    def take(self, grp):
        if not self.own:
            return np.stack([self.rngs[a].standard_normal(self.d) for a in grp])
        empty = grp[self.ptr[grp] >= self.K]
        if empty.size:  # refill (many escapes / redraws): the next block of each stream
            if self.state is not None:
                rows = np.ascontiguousarray(empty, dtype=np.int64)
                blk = np.empty((rows.size, self.K, self.d))
                self._draw(rows, rows.size, blk)
                self.buf[rows] = blk
            else:
                for a in empty:
                    self.buf[a] = self.rngs[a].standard_normal((self.K, self.d))
            self.ptr[empty] = 0
        z = self.buf[grp, self.ptr[grp]]
        self.ptr[grp] += 1
        return z


def descent_batch(ns: NodeSet, starts, seed: int = 0, stats: RaycastStats = None,
                  rngs=None):
    """Many descents at once; the same RNG streams and sigma as calling
    :func:`descent` with ``stream(seed, "descent", s)`` for every start
    (graph.py:46-85), with the Gram-Schmidt projections vectorised over the
    starts of a level and one GPU RayCast launch per level.

    Returns (sigma (S, d+1) int32, r (S, d) fp64)."""
    pts = ns.points
    d = ns.dim
    starts = np.asarray([int(s) for s in starts], dtype=np.int64)
    S = len(starts)
    draws = _Draws(rngs, seed, starts, d)
    sig = np.full((S, d + 1), -1, dtype=np.int64)
    sig[:, 0] = starts
    k = np.ones(S, dtype=np.int64)          # |sigma|
    rr = pts[starts].astype(np.float64).copy()
    fails = np.zeros(S, dtype=np.int64)
    active = np.arange(S)
    while active.size:
        # one direction per active start, drawn from its own stream in the
        # reference order (redraw while the projection vanishes).  The level
        # of every active start is snapshotted: starts advanced while this
        # round's groups are processed must not be picked up again with a
        # direction drawn for their previous level.
        k_act = k[active].copy()
        levels = np.unique(k_act)
        # one draw per active start from its own stream (stream order is per
        # start, so drawing level group by level group is the same draw)
        z = np.empty((active.size, d))
        for kk in levels:
            grp = active[k_act == kk]
            z[np.searchsorted(active, grp)] = draws.take(grp)
        # Gram-Schmidt basis of each start's sigma rows and the projection of
        # its draw, one GPU thread per start (vr_descent_directions; the
        # numpy restatement _mgs_batch / _project_out_batch below serves the
        # rare redraws)
        v, nrm, bad = _descent_directions(ns, sig[active], k_act, z)
        if bad.any():
            a = active[np.argmax(bad)]
            raise DegenerateConfiguration(
                f"generators are affinely dependent (descent from node {int(starts[a])})")
        for m in np.nonzero(nrm < 1e-9)[0]:  # free redraws (graph.py:72-74)
            a, kk = active[m], int(k_act[m])
            diffs = pts[sig[a, 1:kk]] - pts[sig[a, 0]]
            bas = _mgs_batch(diffs[None]) if kk > 1 else np.zeros((1, 0, d))
            while True:
                vv = _project_out_batch(draws.take(np.array([a])), bas)[0]
                if np.linalg.norm(vv) >= 1e-9:
                    v[m] = vv
                    nrm[m] = np.linalg.norm(vv)
                    break
        u = v / nrm[:, None]
        still = []
        # one RayCast for the whole round: eta is padded with copies of its
        # first entry g (thr is a max over eta and g = eta[0], so the padded
        # query is the same query), instead of one launch + sync per level
        kmax = int(k_act.max())
        eta = np.repeat(sig[active, :1], kmax, axis=1)
        for kk in levels:
            eta[k_act == kk, :kk] = sig[active[k_act == kk], :kk]
        res = raycast_batch(ns, rr[active], u, eta.astype(np.int32), stats=stats)
        idx_all, _, rp_all, flag_all = res.to_host()
        for kk in levels:
            sel = k_act == kk
            grp = active[sel]
            idx, rp, flag = idx_all[sel], rp_all[sel], flag_all[sel]
            esc = flag == 1
            if (flag == 3).any():
                raise DegenerateConfiguration(
                    f"degenerate raycast during descent from node {int(starts[grp[np.argmax(flag == 3)]])}")
            fails[grp[esc]] += 1
            if (fails[grp[esc]] >= DESCENT_RETRIES).any():
                a = grp[esc][np.argmax(fails[grp[esc]] >= DESCENT_RETRIES)]
                raise RetryExhausted(f"descent from node {int(starts[a])} stuck at level {kk}")
            still.append(grp[esc])
            ok = ~esc
            g_ok = grp[ok]
            if g_ok.size:
                new = np.sort(np.concatenate([sig[g_ok, :kk], idx[ok, None].astype(np.int64)], 1), 1)
                sig[g_ok, :kk + 1] = new
                k[g_ok] = kk + 1
                rr[g_ok] = rp[ok]
                fails[g_ok] = 0
                if kk + 1 < d + 1:
                    still.append(g_ok)
        active = np.sort(np.concatenate(still)) if still else np.zeros(0, dtype=np.int64)
    return sig.astype(np.int32), rr


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
    """Vertex, edge-consistency and (small instances) oracle checks
    (graph.py:202-245), on the device: verify_vertices over every vertex,
    then the incidence count of every recorded edge (vr_edge_incidence /
    vr_edge_check) against its recorded count -- an interior edge (count 2)
    must have exactly two incident vertices, whose sigmas then intersect in
    eta; a boundary edge (count 1) exactly one.  Only failures are brought
    to the host."""
    ns = mesh.nodes
    dev = ns.device_records()[0].device
    d = ns.dim
    dv = mesh.device_arrays()
    a = None if dv is not None else mesh.arrays()
    if dv is not None:
        sig_d, r_d, ek_d, ec_d = dv["sigma"], dv["r"], dv["edge_key"], dv["edge_count"]
    else:
        sig_d = torch.as_tensor(a["sigma"], device=dev)
        r_d = torch.as_tensor(a["r"], device=dev)
        ek_d = torch.as_tensor(a["edge_key"], device=dev)
        ec_d = torch.as_tensor(a["edge_count"], device=dev)
    # the reference-style dict views, once materialised, are what a caller
    # edits (mesh.vertices[sigma] = ...): verify what they hold
    if mesh._vertices is not None:
        keys = list(mesh._vertices)
        sig_d = torch.as_tensor(np.array(keys, dtype=np.int32).reshape(-1, d + 1), device=dev)
        r_d = torch.as_tensor(np.array([mesh._vertices[k].r for k in keys],
                                       dtype=np.float64).reshape(-1, d), device=dev)
    if mesh._edge_counts is not None:
        ek_d = torch.as_tensor(np.array(list(mesh._edge_counts), dtype=np.int32).reshape(-1, d),
                               device=dev)
        ec_d = torch.as_tensor(np.array(list(mesh._edge_counts.values()), dtype=np.int32),
                               device=dev)
    nv = int(sig_d.shape[0])
    report = VerifyReport(vertices_total=nv)
    if nv:
        ok = verify_vertices_device(ns, sig_d, r_d)
        bad = torch.nonzero(~ok).flatten().cpu().numpy()
        sig_bad = sig_d[torch.as_tensor(bad, device=dev)].cpu().numpy() if bad.size else []
        report.vertex_failures = [tuple(int(x) for x in s) for s in sig_bad]
    if ek_d.shape[0]:
        ikeys, icnt = edge_incidence(ns, sig_d)
        inc = torch.empty(ek_d.shape[0], dtype=torch.int32, device=dev)
        ek32 = ek_d.to(torch.int32).contiguous()
        _lib.check(_lib.lib().vr_edge_check(_lib.ptr(ikeys), _lib.ptr(icnt), ikeys.shape[0],
                                            _lib.ptr(ek32), ek32.shape[0], ns.dim, _lib.ptr(inc),
                                            _lib.stream_handle()), "vr_edge_check")
        ec = ec_d.to(torch.int32)
        fail = ((ec != 1) & (ec != 2)) | (inc != ec)
        idx = torch.nonzero(fail).flatten()
        if idx.numel():
            keys = ek32[idx].cpu().numpy()
            cs, ks = ec[idx].cpu().numpy(), inc[idx].cpu().numpy()
            for key, c, k in zip(keys, cs, ks):
                eta = tuple(int(x) for x in key)
                if c in (1, 2):
                    report.edge_failures.append((eta, f"count {int(c)} but {int(k)} vertices"))
                else:
                    report.edge_failures.append((eta, f"invalid count {int(c)}"))
    if oracle is None:
        oracle = ns.dim <= 3 and ns.n <= 200
    if oracle:
        report.oracle_checked = True
        truth = brute_force_vertices(ns)
        verts = mesh.vertices
        ours = {s: v.r for s, v in verts.items()}
        report.oracle_missing = sorted(set(truth) - set(ours))
        report.oracle_extra = sorted(set(ours) - set(truth))
        for s in set(truth) & set(ours):
            if np.linalg.norm(truth[s] - ours[s]) > coord_tol * max(1.0, float(np.linalg.norm(truth[s]))):
                report.oracle_coord_failures.append(s)
    return report


# ---------------------------------------------------------------------------
# level-synchronous device traversal (csrc/traverse.cu)
# ---------------------------------------------------------------------------

class _Tables(ctypes.Structure):
    _fields_ = [("vkeys", ctypes.c_void_p), ("vstate", ctypes.c_void_p),
                ("vval", ctypes.c_void_p), ("vlevel", ctypes.c_void_p),
                ("vcap", ctypes.c_int64), ("ekeys", ctypes.c_void_p),
                ("estate", ctypes.c_void_p), ("ecount", ctypes.c_void_p),
                ("ecap", ctypes.c_int64), ("overflow", ctypes.c_void_p)]


class _RunState(ctypes.Structure):  # vr_trav_state
    _fields_ = [("vsig", ctypes.c_void_p), ("vr", ctypes.c_void_p), ("vcap_arrays", ctypes.c_int64),
                ("bsig", ctypes.c_void_p), ("bu", ctypes.c_void_p), ("bcap", ctypes.c_int64),
                ("nv", ctypes.c_int64), ("nb", ctypes.c_int64), ("e_ub", ctypes.c_int64),
                ("f0", ctypes.c_int64), ("f1", ctypes.c_int64), ("level", ctypes.c_int32),
                ("phase", ctypes.c_int32), ("pending_rays", ctypes.c_int64),
                ("n_new", ctypes.c_int64), ("n_esc", ctypes.c_int64),
                ("n_degenerate", ctypes.c_int64), ("n_bad", ctypes.c_int64),
                ("overflow", ctypes.c_int64), ("rays", ctypes.c_int64), ("need", ctypes.c_int32),
                ("need_amount", ctypes.c_int64), ("sub_n", ctypes.c_int32),
                ("sub_j", ctypes.c_int32)]


RUN_DONE, RUN_NEED_WS, RUN_NEED_V, RUN_NEED_E, RUN_NEED_B, RUN_ERROR = range(6)


def _pow2(n):
    return 1 << max(10, int(n - 1).bit_length())


def _excl_cumsum(x):
    """Exclusive prefix sum (int64) and the total, on the device."""
    c = torch.cumsum(x, 0, dtype=torch.int64)
    return c - x.to(torch.int64), c


class DeviceTraversal:
    """Device state of one traversal: vertex / edge hash tables, vertex,
    boundary arrays.  Capacities grow geometrically between levels."""

    def __init__(self, ns: NodeSet, vcap_hint=None, ecap_hint=None):
        rec, sqmax = ns.device_records()
        self.ns, self.rec, self.sqmax, self.dev = ns, rec, sqmax, rec.device
        self.d = ns.dim
        self.L = _lib.lib()
        d = self.d
        vcap = _pow2(vcap_hint or 4 * max(1024, ns.n))
        self.overflow = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self._alloc_vtable(vcap)
        self._alloc_etable(_pow2(ecap_hint or 2 * vcap))
        self.vsig = torch.empty((vcap // 2, d + 1), dtype=torch.int32, device=self.dev)
        self.vr = torch.empty((vcap // 2, d), dtype=torch.float64, device=self.dev)
        self.bsig = torch.empty((1024, d + 1), dtype=torch.int32, device=self.dev)
        self.bu = torch.empty((1024, d), dtype=torch.float64, device=self.dev)
        self.nv = 0
        self.nb = 0
        self.e_ub = 0
        self.work = None  # optional VR_WORK_COUNTERS tensor (pruned-kernel accounting)
        # native level driver (csrc/level.cu) unless VR_NATIVE_LEVEL=0
        self.native = os.environ.get("VR_NATIVE_LEVEL", "1") != "0" and ns.fast_paths

    def _alloc_vtable(self, cap):
        d = self.d
        self.vkeys = torch.empty(cap * (d + 1), dtype=torch.int32, device=self.dev)
        self.vstate = torch.zeros(cap, dtype=torch.int32, device=self.dev)
        self.vval = torch.empty(cap, dtype=torch.int32, device=self.dev)
        self.vlevel = torch.empty(cap, dtype=torch.int32, device=self.dev)
        self.vcap = cap

    def _alloc_etable(self, cap):
        self.ekeys = torch.empty(cap * self.d, dtype=torch.int32, device=self.dev)
        # (state, count) pairs of the slots interleaved: ecount == estate + 1 tells
        # the library, and a slot's state and counter share one 32-B sector
        self.epairs = torch.zeros(2 * cap, dtype=torch.int32, device=self.dev)
        self.estate = self.epairs[0::2]
        self.ecount = self.epairs[1::2]
        self.ecap = cap

    def tables(self):
        p = _lib.ptr
        return _Tables(p(self.vkeys).value, p(self.vstate).value, p(self.vval).value,
                       p(self.vlevel).value, self.vcap, p(self.ekeys).value,
                       p(self.estate).value, p(self.ecount).value, self.ecap,
                       p(self.overflow).value)

    def _sh(self):
        return _lib.stream_handle()

    def ensure_vertices(self, extra):
        """Room for `extra` more vertices in the arrays and the hash set."""
        need = self.nv + extra
        if need > self.vsig.shape[0]:
            cap = max(need, 2 * self.vsig.shape[0])
            self.vsig = torch.cat([self.vsig[:self.nv],
                                   torch.empty((cap - self.nv, self.d + 1), dtype=torch.int32,
                                               device=self.dev)])
            self.vr = torch.cat([self.vr[:self.nv],
                                 torch.empty((cap - self.nv, self.d), dtype=torch.float64,
                                             device=self.dev)])
        if 2 * need > self.vcap:
            self._alloc_vtable(_pow2(2 * need))  # load <= 0.5
            T = self.tables()
            _lib.check(self.L.vr_trav_insert_vertices(ctypes.byref(T), self.d,
                                                      _lib.ptr(self.vsig), self.nv, 0, -1, 0,
                                                      self._sh()), "rehash vertices")

    def ensure_edges(self, extra):
        if 2 * (self.e_ub + extra) > self.ecap:
            ok, os_, oc, ocap = self.ekeys, self.estate, self.ecount, self.ecap
            # e_ub counts every (vertex, edge) incidence, about twice the
            # distinct edges, so 2x keeps the real load near 0.25 (4x made
            # config 5's table 2^31 slots, 86 GB)
            self._alloc_etable(_pow2(2 * (self.e_ub + extra)))
            T = self.tables()
            _lib.check(self.L.vr_trav_rehash_edges(ctypes.byref(T), self.d, _lib.ptr(ok),
                                                   _lib.ptr(os_), _lib.ptr(oc), ocap,
                                                   self._sh()), "rehash edges")

    def ensure_boundary(self, extra):
        need = self.nb + extra
        if need > self.bsig.shape[0]:
            cap = max(need, 2 * self.bsig.shape[0])
            self.bsig = torch.cat([self.bsig[:self.nb],
                                   torch.empty((cap - self.nb, self.d + 1), dtype=torch.int32,
                                               device=self.dev)])
            self.bu = torch.cat([self.bu[:self.nb],
                                 torch.empty((cap - self.nb, self.d), dtype=torch.float64,
                                             device=self.dev)])

    def seed_vertex(self, sigma):
        """Insert the descent vertex (level 0) with its fp64 circumcentre."""
        self.seed_vertices(np.asarray(sigma, dtype=np.int32)[None])

    def seed_vertices(self, sigmas):
        """Insert distinct seed vertices (sorted sigma rows) at level 0."""
        sig = np.ascontiguousarray(sigmas, dtype=np.int32).reshape(-1, self.d + 1)
        m = sig.shape[0]
        self.ensure_vertices(m)
        self.ensure_edges((self.d + 1) * m)
        s = torch.as_tensor(sig, device=self.dev)
        self.vsig[0:m] = s
        ok = torch.empty(m, dtype=torch.uint8, device=self.dev)
        _lib.check(self.L.vr_circumcenters(_lib.ptr(self.rec), self.d, _lib.ptr(s), m,
                                           _lib.ptr(self.vr), _lib.ptr(ok), self._sh()),
                   "vr_circumcenters")
        if not bool(ok.all()):
            raise DegenerateConfiguration("a seed vertex has an affinely dependent sigma")
        T = self.tables()
        _lib.check(self.L.vr_trav_insert_vertices(ctypes.byref(T), self.d, _lib.ptr(s), m, 0, 0,
                                                  1, self._sh()), "insert seeds")
        self.nv = m
        self.e_ub = (self.d + 1) * m

    def _raycast(self, rx, ru, reta, stats, ws):
        res = raycast_batch(self.ns, rx, ru, reta, want_rp=False, stats=stats, workspace=ws,
                            work=self.work)
        return res.idx, res.flag

    def _level_native(self, f0, f1, lvl, stats, ws):
        """level() through the native driver (csrc/level.cu): two C-ABI calls
        and two synchronisations instead of ~40 torch / ctypes operations."""
        d, L, dev, sh = self.d, self.L, self.dev, self._sh()
        ws = ws if ws is not None else Workspace()
        F = f1 - f0
        fs = self.vsig[f0:f1]
        fr = self.vr[f0:f1]
        p = _lib.ptr
        open_mask = ws.get("lv_open_mask", (F, d + 1), torch.uint8, dev)
        open_cnt = ws.get("lv_open_cnt", (F,), torch.int32, dev)
        off = ws.get("lv_open_off", (F,), torch.int64, dev)
        T = self.tables()
        nr = ctypes.c_int64(0)
        wsb = ctypes.c_int64(0)
        _lib.check(L.vr_trav_level_workspace(F, 0, self.ns.n, d, ctypes.byref(wsb)),
                   "level_workspace")
        scratch = ws.get("lv_scratch", (wsb.value,), torch.uint8, dev)
        _lib.check(L.vr_trav_level_open(ctypes.byref(T), d, p(fs), F, p(open_mask), p(open_cnt),
                                        p(off), ctypes.byref(nr), p(scratch), scratch.numel(), sh),
                   "level_open")
        R = int(nr.value)
        if R == 0:
            return 0
        if stats is not None:
            stats.add(R)
        rx = ws.get("lv_rx", (R, d), torch.float64, dev)
        ru = ws.get("lv_ru", (R, d), torch.float64, dev)
        reta = ws.get("lv_reta", (R, d), torch.int32, dev)
        rpar = ws.get("lv_rpar", (R,), torch.int32, dev)
        hidx = ws.get("lv_hidx", (R,), torch.int32, dev)
        ht = ws.get("lv_ht", (R,), torch.float64, dev)
        hflag = ws.get("lv_hflag", (R,), torch.uint8, dev)
        bad = ws.get("lv_bad", (2,), torch.int32, dev)
        self.ensure_vertices(R)
        T = self.tables()
        rsig = ws.get("lv_rsig", (R, d + 1), torch.int32, dev)
        slot = ws.get("lv_slot", (R,), torch.int64, dev)
        newf = ws.get("lv_newf", (R,), torch.int32, dev)
        escf = ws.get("lv_escf", (R,), torch.int32, dev)
        noff = ws.get("lv_noff", (R,), torch.int64, dev)
        eoff = ws.get("lv_eoff", (R,), torch.int64, dev)
        counts = np.zeros(5, dtype=np.int64)
        ns = self.ns
        ix = ns.prune_index(dev)
        s32 = ns.screen32(dev)
        _lib.check(L.vr_trav_level_workspace(F, R, ns.n, d, ctypes.byref(wsb)), "level_workspace")
        scratch = ws.get("lv_scratch", (wsb.value,), torch.uint8, dev)
        _lib.check(L.vr_trav_level_cast(
            ctypes.byref(T), p(self.rec), ns.n, d, self.sqmax, ctypes.byref(s32.struct),
            ctypes.byref(ix.struct), p(fs), p(fr), F, p(open_mask), p(off), R, lvl, p(rx), p(ru),
            p(reta), p(rpar), p(hidx), p(ht), p(hflag), p(rsig), p(slot), p(newf), p(escf),
            p(noff), p(eoff), p(bad), p(self.work), counts.ctypes.data, p(scratch),
            scratch.numel(), sh), "level_cast")
        n_new, n_esc, n_deg, n_bad, ovf = (int(v) for v in counts)
        if n_bad:
            raise DegenerateConfiguration("generators of a frontier vertex are affinely dependent")
        if n_deg:
            raise DegenerateConfiguration(
                f"{n_deg} edge raycasts hit a generator on the circumsphere band")
        if ovf:
            raise RuntimeError("traversal hash table overflow")
        self.ensure_edges((d + 1) * n_new)
        T = self.tables()
        _lib.check(L.vr_trav_finalize(ctypes.byref(T), p(self.rec), d, p(rsig), p(slot),
                                      p(newf), p(noff), R, f1, p(self.vsig), p(self.vr),
                                      p(bad[1:]), 1, sh), "finalize")
        self.e_ub += (d + 1) * n_new
        if n_esc:
            self.ensure_boundary(n_esc)
            _lib.check(L.vr_trav_boundary(d, p(escf), p(eoff), p(rpar), p(ru), R, p(fs), self.nb,
                                          p(self.bsig), p(self.bu), sh), "boundary")
            self.nb += n_esc
        self.nv = f1 + n_new
        self.rays_last = R
        return n_new

    def run(self, f0, f1, first_level, last_level=-1, stats=None, ws=None):
        """Levels first_level .. last_level (-1: until done) natively
        (vr_trav_run: the level loop in C++, two synchronisations per level,
        no per-level host work); returns the new-vertex count per level.
        Capacities grow here when the driver asks for them."""
        d, L, p = self.d, self.L, _lib.ptr
        ws = ws if ws is not None else Workspace()
        ns = self.ns
        ix, s32 = ns.prune_index(self.dev), ns.screen32(self.dev)
        cap = 4096
        level_new = np.zeros(cap, dtype=np.int64)
        S = _RunState()
        S.nv, S.nb, S.e_ub = self.nv, self.nb, self.e_ub
        S.f0, S.f1, S.level, S.phase = f0, f1, first_level, 0
        wsb = 0
        scratch = None
        while True:
            S.vsig, S.vr, S.vcap_arrays = p(self.vsig).value, p(self.vr).value, self.vsig.shape[0]
            S.bsig, S.bu, S.bcap = p(self.bsig).value, p(self.bu).value, self.bsig.shape[0]
            T = self.tables()
            _lib.check(L.vr_trav_run(ctypes.byref(T), ctypes.byref(S), p(self.rec), ns.n, d,
                                     self.sqmax, ctypes.byref(s32.struct), ctypes.byref(ix.struct),
                                     int(last_level), level_new.ctypes.data, cap, p(self.work),
                                     p(scratch), wsb, _lib.stream_handle()), "vr_trav_run")
            need, amt = int(S.need), int(S.need_amount)
            if need == RUN_DONE:
                break
            if need == RUN_NEED_WS:
                old = scratch
                scratch = ws.get("run_scratch", (int(1.25 * amt) + 4096,), torch.uint8, self.dev)
                if old is not None and int(S.phase) == 2 and scratch.data_ptr() != old.data_ptr():
                    # the level's open step is done: its result is the prefix
                    scratch[:old.numel()].copy_(old)
                wsb = scratch.numel()
            elif need == RUN_NEED_V:
                self.nv = int(S.nv)
                self.ensure_vertices(amt - self.nv)
            elif need == RUN_NEED_E:
                self.e_ub = int(S.e_ub)
                self.ensure_edges(amt - self.e_ub)
            elif need == RUN_NEED_B:
                self.nb = int(S.nb)
                self.ensure_boundary(amt - self.nb)
            else:
                if S.n_bad:
                    raise DegenerateConfiguration(
                        "generators of a frontier vertex are affinely dependent")
                if S.n_degenerate:
                    raise DegenerateConfiguration(
                        f"{int(S.n_degenerate)} edge raycasts hit a generator on the circumsphere band")
                raise RuntimeError("traversal hash table overflow")
        self.nv, self.nb, self.e_ub = int(S.nv), int(S.nb), int(S.e_ub)
        if stats is not None:
            stats.add(int(S.rays))
        self.rays_last = int(S.rays)
        return [int(v) for v in level_new[first_level:int(S.level)]], int(S.f0), int(S.f1)

    def level(self, f0, f1, lvl, stats=None, ws=None, raycast_fn=None):
        """Expand frontier vertices [f0, f1); returns the number of new vertices.

        raycast_fn(x, u, eta) -> (idx int32, flag uint8) replaces the local
        fused RayCast (parallel.ShardedRaycast splits the level's rays across
        ranks and all-gathers the hits)."""
        if raycast_fn is None and self.native and self.ns.n >= PRUNE_MIN_GENERATORS:
            return self._level_native(f0, f1, lvl, stats, ws)
        d, L, dev, sh = self.d, self.L, self.dev, self._sh()
        F = f1 - f0
        fs = self.vsig[f0:f1]
        fr = self.vr[f0:f1]
        open_mask = torch.empty((F, d + 1), dtype=torch.uint8, device=dev)
        open_cnt = torch.empty(F, dtype=torch.int32, device=dev)
        T = self.tables()
        _lib.check(L.vr_trav_open_edges(ctypes.byref(T), d, _lib.ptr(fs), F, _lib.ptr(open_mask),
                                        _lib.ptr(open_cnt), sh), "open_edges")
        off, inc = _excl_cumsum(open_cnt)
        R = int(inc[-1].item())
        if R == 0:
            return 0
        rx = torch.empty((R, d), dtype=torch.float64, device=dev)
        ru = torch.empty((R, d), dtype=torch.float64, device=dev)
        reta = torch.empty((R, d), dtype=torch.int32, device=dev)
        rpar = torch.empty(R, dtype=torch.int32, device=dev)
        bad = torch.zeros(2, dtype=torch.int32, device=dev)
        _lib.check(L.vr_trav_emit_rays(_lib.ptr(self.rec), d, _lib.ptr(fs), _lib.ptr(fr), F,
                                       _lib.ptr(open_mask), _lib.ptr(off), _lib.ptr(rx),
                                       _lib.ptr(ru), _lib.ptr(reta), _lib.ptr(rpar),
                                       _lib.ptr(bad), sh), "emit_rays")
        if raycast_fn is None:
            hit_idx, hit_flag = self._raycast(rx, ru, reta, stats, ws)
        else:
            hit_idx, hit_flag = raycast_fn(rx, ru, reta)
        self.ensure_vertices(R)
        T = self.tables()
        rsig = torch.empty((R, d + 1), dtype=torch.int32, device=dev)
        slot = torch.empty(R, dtype=torch.int64, device=dev)
        newf = torch.empty(R, dtype=torch.int32, device=dev)
        escf = torch.empty(R, dtype=torch.int32, device=dev)
        _lib.check(L.vr_trav_claim(ctypes.byref(T), d, _lib.ptr(reta), _lib.ptr(hit_idx),
                                   _lib.ptr(hit_flag), R, lvl, _lib.ptr(rsig), _lib.ptr(slot),
                                   _lib.ptr(newf), _lib.ptr(escf), sh), "claim")
        noff, ninc = _excl_cumsum(newf)
        eoff, einc = _excl_cumsum(escf)
        ndeg = (hit_flag == 3).sum()
        summary = torch.stack([ninc[-1], einc[-1], ndeg.to(torch.int64), bad[0].to(torch.int64),
                               self.overflow[0].to(torch.int64)]).cpu().numpy()
        n_new, n_esc, n_deg, n_bad, ovf = (int(v) for v in summary)
        if n_bad:
            raise DegenerateConfiguration("generators of a frontier vertex are affinely dependent")
        if n_deg:
            raise DegenerateConfiguration(
                f"{n_deg} edge raycasts hit a generator on the circumsphere band")
        if ovf:
            raise RuntimeError("traversal hash table overflow")
        self.ensure_edges((d + 1) * n_new)
        T = self.tables()
        _lib.check(L.vr_trav_finalize(ctypes.byref(T), _lib.ptr(self.rec), d, _lib.ptr(rsig),
                                      _lib.ptr(slot), _lib.ptr(newf), _lib.ptr(noff), R, f1,
                                      _lib.ptr(self.vsig), _lib.ptr(self.vr), _lib.ptr(bad[1:]),
                                      1, sh), "finalize")
        self.e_ub += (d + 1) * n_new
        if n_esc:
            self.ensure_boundary(n_esc)
            _lib.check(L.vr_trav_boundary(d, _lib.ptr(escf), _lib.ptr(eoff), _lib.ptr(rpar),
                                          _lib.ptr(ru), R, _lib.ptr(fs), self.nb,
                                          _lib.ptr(self.bsig), _lib.ptr(self.bu), sh), "boundary")
            self.nb += n_esc
        self.nv = f1 + n_new
        self.rays_last = R
        return n_new

    def edges(self):
        """Published edge keys and counts (device tensors, hash-table order):
        two native passes over the slot states (vr_trav_edges_count /
        vr_trav_edges_compact)."""
        T = self.tables()
        nbytes = ctypes.c_int64(0)
        _lib.check(self.L.vr_trav_edges_count(ctypes.byref(T), None, None, None,
                                              ctypes.byref(nbytes), None), "edges_count (size)")
        nc = (self.ecap + 4095) // 4096
        off = torch.empty(nc + 1, dtype=torch.int64, device=self.dev)
        tmp = torch.empty(max(1, nbytes.value), dtype=torch.uint8, device=self.dev)
        ne = ctypes.c_int64(0)
        _lib.check(self.L.vr_trav_edges_count(ctypes.byref(T), _lib.ptr(off), ctypes.byref(ne),
                                              _lib.ptr(tmp), ctypes.byref(nbytes), self._sh()),
                   "edges_count")
        keys = torch.empty((ne.value, self.d), dtype=torch.int32, device=self.dev)
        cnt = torch.empty(ne.value, dtype=torch.int32, device=self.dev)
        slots = torch.empty(max(1, ne.value), dtype=torch.int64, device=self.dev)
        _lib.check(self.L.vr_trav_edges_compact(ctypes.byref(T), self.d, _lib.ptr(off), ne.value,
                                                _lib.ptr(slots), _lib.ptr(keys), _lib.ptr(cnt),
                                                self._sh()), "edges_compact")
        return keys, cnt  # hash order; Mesh sorts lexicographically on materialisation


def _level_raycaster(ns, stats, group, work=None):
    """None (local fused RayCast) or a ShardedRaycast over the ranks of the
    default / given process group (`work`: this rank's kernel work counters)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return None
    from .parallel import ShardedRaycast

    def fn(x, u, eta):
        r = raycast_batch(ns, x, u, eta, want_rp=False, stats=stats, work=work)
        return r.idx, r.flag

    return ShardedRaycast(fn, group)


def _table_estimate(ns, v_guess):
    """Vertex count the traversal tables are pre-sized for: the Poisson
    estimate, capped by C(N, d+1) and by a quarter of the free device memory
    (~(d+1)(4d + 28) + 8d bytes per vertex of tables and arrays); the tables
    still grow geometrically past it, so the cap only bounds the up-front
    allocation of small high-d inputs."""
    from math import comb
    d = ns.dim
    v = min(int(v_guess), comb(ns.n, d + 1), 1 << 26)
    try:
        free, _ = torch.cuda.mem_get_info(ns.device_records()[0].device)
        per_vertex = (d + 1) * (4 * d + 28) + 8 * d + 16 * (d + 1)
        v = min(v, max(1 << 12, free // 4 // per_vertex))
    except RuntimeError:
        pass
    return max(int(v), 1)


def _group_size(group):
    import torch.distributed as dist
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def _sharding():
    """Multi-rank traversal scheme: "owner" (default; parallel.ShardedTraversal,
    owner-sharded tables, per-level all-to-all) or "replicated" (replicated
    tables, ray-sharded levels, one all-gather of the hits per level)."""
    mode = os.environ.get("VR_SHARDING", "owner")
    if mode not in ("owner", "replicated"):
        raise ValueError(f"VR_SHARDING must be owner or replicated, got {mode!r}")
    return mode


def set_sub_rounds(rays_per_round: int = -1, max_rounds: int = -1):
    """Sub-rounds of large traversal levels (vr_trav_set_sub_rounds): a level
    whose frontier would cast more than ``rays_per_round`` rays is cast in up
    to ``max_rounds`` interleaved rounds, so that vertices found by an earlier
    round close the edges later rounds would have cast again (the reference's
    one-vertex-at-a-time loop never casts them, graph.py:115-128).  0 = never
    split; -1, -1 = the library defaults (VR_SUB_RAYS / VR_SUB_MAX).  The mesh
    (vertex set, edges, boundary rays) does not depend on the setting."""
    _lib.check(_lib.lib().vr_trav_set_sub_rounds(int(rays_per_round), int(max_rounds)),
               "vr_trav_set_sub_rounds")


def voronoi_graph(ns: NodeSet, seed: int = 0, *, method: str = "incircle_heuristic",
                  eps: float = None, stats: RaycastStats = None, return_info: bool = False,
                  group=None, work=None):
    """Full Voronoi mesh by exhaustive edge-tracked traversal (graph.py:88-146).

    Level-synchronous on the device: every level raycasts all open edges of
    the frontier in one fused launch.  The vertex set, edge counts and the
    boundary-ray multiset equal the reference's depth-first result; vertex
    coordinates are fp64 circumcentres of sigma.
    """
    _resolve_raycaster(method, eps)
    if stats is None:
        stats = RaycastStats()
    first = descent(ns, 0, _rng.stream(seed, "descent", 0), stats)
    # size the tables for the expected diagram (mean Voronoi vertices per
    # generator of a Poisson diagram in d dimensions) so that they rarely
    # grow: config 3 rehashed its edge table 8 times from the default size
    vpg = {2: 2, 3: 7, 4: 32, 5: 190, 6: 1300, 7: 9000, 8: 66000}.get(ns.dim, 4)
    v_est = _table_estimate(ns, ns.n * vpg)
    size = _group_size(group)
    if size > 1 and _sharding() == "owner" and ns.fast_paths:
        from .parallel import DeviceShardOps, ShardedTraversal
        share = v_est // size + 1024
        st = ShardedTraversal(ns, DeviceShardOps(ns, vcap_hint=max(4096, 2 * share),
                                                 ecap_hint=2 * (ns.dim + 1) * share), group)
        st.ops.work = work
        st.seed(np.asarray([first.sigma], dtype=np.int32))
        levels, lvl = [], 1
        while True:
            n_new = st.level(lvl, stats)
            levels.append(n_new)
            if n_new == 0:
                break
            lvl += 1
        mesh = st.gather()
        if return_info:
            return mesh, {"levels": levels, "vertices": mesh.n_vertices,
                          "boundary": int(mesh.device_arrays()["boundary_sigma"].shape[0]),
                          "sharding": "owner"}
        return mesh
    tr = DeviceTraversal(ns, vcap_hint=max(4 * ns.n, 2 * v_est),
                         ecap_hint=2 * (ns.dim + 1) * v_est)
    tr.work = work
    tr.seed_vertex(first.sigma)
    from .raycast import Workspace
    ws = Workspace()
    f0, f1, lvl = 0, 1, 1
    levels = []
    rfn = _level_raycaster(ns, stats, group, tr.work)
    if rfn is None and tr.native and ns.n >= PRUNE_MIN_GENERATORS:
        news, _, _ = tr.run(0, 1, 1, -1, stats=stats, ws=ws)  # the native level loop
        sizes = [1] + news
        levels = [(sizes[k], news[k]) for k in range(len(news))]
        f0 = f1 = tr.nv
    while f1 > f0:
        n_new = tr.level(f0, f1, lvl, stats=stats, ws=ws, raycast_fn=rfn)
        levels.append((f1 - f0, n_new))
        f0, f1, lvl = f1, f1 + n_new, lvl + 1
    ek, ec = tr.edges()
    mesh = Mesh.from_device(ns, tr.vsig[:tr.nv], tr.vr[:tr.nv], ek, ec, tr.bsig[:tr.nb],
                            tr.bu[:tr.nb])
    if return_info:
        return mesh, {"levels": levels, "vertices": tr.nv, "boundary": tr.nb}
    return mesh


def voronoi_local(ns: NodeSet, starts, hops: int, seed: int = 0, stats: RaycastStats = None,
                  return_levels: bool = False, group=None, work=None):
    """All Voronoi vertices within `hops` edge hops of the descent vertices of
    `starts` (SURVEY.md §8(d) config 5 "local traversal").

    The seed vertices come from the reference descent with the streams
    ``stream(seed, "descent", s)`` (graph.py:46-85); the level-synchronous
    traversal then runs `hops` levels.  BFS level = hop distance, so the
    result is the union of the L-hop balls, independent of visiting order.
    Returns a Mesh (and, with return_levels, the hop level of every vertex).
    """
    if stats is None:
        stats = RaycastStats()
    import torch.distributed as dist
    size = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if size > 1:
        # each rank descends its contiguous share of the starts (every start
        # has its own stream, so the result does not depend on the sharding);
        # one all-gather of the sigmas
        from .parallel import allgather_rows, shard_bounds
        starts = np.asarray([int(s) for s in starts], dtype=np.int64)
        lo, hi = shard_bounds(len(starts), size, dist.get_rank(group))
        part, _ = descent_batch(ns, starts[lo:hi], seed=seed, stats=stats)
        dev = ns.device_records()[0].device
        sig = allgather_rows(torch.as_tensor(part.reshape(-1, ns.dim + 1), device=dev),
                             group).cpu().numpy()
    else:
        sig, _ = descent_batch(ns, starts, seed=seed, stats=stats)
    _, first = np.unique(sig, axis=0, return_index=True)
    sig = sig[np.sort(first)]
    if size > 1 and _sharding() == "owner" and ns.fast_paths:
        from .parallel import DeviceShardOps, ShardedTraversal
        share = 6 * len(sig) * 4 ** min(hops, 8) // size + 1024
        st = ShardedTraversal(ns, DeviceShardOps(ns, vcap_hint=max(4096, share)), group)
        st.ops.work = work
        st.seed(sig)
        for lvl in range(1, hops + 1):
            if st.level(lvl, stats) == 0:
                break
        return st.gather(with_levels=True) if return_levels else st.gather()
    tr = DeviceTraversal(ns, vcap_hint=max(4 * ns.n, 6 * len(sig) * 4 ** min(hops, 8)))
    tr.work = work
    tr.seed_vertices(sig)
    from .raycast import Workspace
    ws = Workspace()
    f0, f1 = 0, tr.nv
    bounds = [(0, f1)]
    rfn = _level_raycaster(ns, stats, group, work)
    if rfn is None and tr.native and ns.n >= PRUNE_MIN_GENERATORS and hops >= 1:
        news, _, _ = tr.run(0, f1, 1, hops, stats=stats, ws=ws)  # the native level loop
        for n_new in news:
            f0, f1 = f1, f1 + n_new
            bounds.append((f0, f1))
        hops = 0
    for lvl in range(1, hops + 1):
        if f1 == f0:
            break
        n_new = tr.level(f0, f1, lvl, stats=stats, ws=ws, raycast_fn=rfn)
        f0, f1 = f1, f1 + n_new
        bounds.append((f0, f1))
    ek, ec = tr.edges()
    mesh = Mesh.from_device(ns, tr.vsig[:tr.nv], tr.vr[:tr.nv], ek, ec, tr.bsig[:tr.nb],
                            tr.bu[:tr.nb])
    if return_levels:
        lv = np.zeros(tr.nv, dtype=np.int8)
        for h, (a, b) in enumerate(bounds):
            lv[a:b] = h
        return mesh, lv
    return mesh
