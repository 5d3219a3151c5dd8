"""Generators, mesh types and vertex checks (drop-in for voronray.core).

Mirrors pkg/src/voronray/core.py: ``NodeSet`` / ``build_node_set`` keep the
reference constructor, validation and errors (core.py:35-57, 145-169); the
nearest-neighbour query (core.py:62-142) and ``verify_vertex``
(core.py:279-296) run on the B200 through the C-ABI library.  The generator
set lives in HBM as 16-B aligned records [x, |x|^2, pad] (one copy per
device, packed on first use).

``Mesh`` is array-backed: the traversal returns sigma /
coordinate / edge / boundary arrays and the reference's dict views
(``vertices``, ``edge_counts``, ``boundary``) are materialised lazily.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from itertools import combinations

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatch, DuplicatePoint

# Reference tolerances (core.py:24-32).
TOL_VERTEX = 1e-8
TOL_DEGENERATE = 1e-10
HALFSPACE_SLACK = 1e-12
_SCAN_MAX = 2048

# d = 2 .. 16: the exhaustive fp64 RayCast, MC and traversal kernels; the
# fp32 / tensor-core screens and the kd-pruned kernels cover d <= 8 (the
# configs' range), so larger d takes the exhaustive fp64 path automatically.
MIN_DIM, MAX_DIM = 2, 16
FAST_MAX_DIM = 8


def _device(device=None):
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError("the B200 kernels need a CUDA device")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


class NodeSet:
    """Immutable generator points, resident in HBM as packed records.

    ``backend`` is accepted for API compatibility ("scan", "kdtree", "auto",
    core.py:52-57); every query is a brute-force scan on the GPU, which is
    the reference's semantic contract (exact equivalence with a linear scan,
    smallest index on ties, core.py:36-42).
    """

    def __init__(self, points, backend="auto"):
        pts = np.array(points, dtype=float, copy=True)
        if pts.ndim != 2:
            raise DimensionMismatch("points must form a 2-d array of shape (n, d)")
        self.points = np.ascontiguousarray(pts)
        self.points.setflags(write=False)
        self.n, self.dim = self.points.shape
        if not MIN_DIM <= self.dim <= MAX_DIM:
            raise DimensionMismatch(
                f"the B200 kernels support {MIN_DIM} <= d <= {MAX_DIM}, got d={self.dim}")
        self._sq = np.einsum("ij,ij->i", self.points, self.points)
        if backend == "auto":
            backend = "scan" if self.n <= _SCAN_MAX else "kdtree"
        if backend not in ("scan", "kdtree"):
            raise ValueError(f"unknown backend {backend!r}")
        self.backend = backend
        self._dev = {}
        self._prune = {}
        self._s32 = {}

    def __len__(self):
        return self.n

    @property
    def stride(self):
        return (self.dim + 2) & ~1

    def device_records(self, device=None):
        """(records tensor (rows, stride) fp64 on `device`, max |x|^2 as float).

        rows = n rounded up to 512; rows >= n are RayCast sentinels."""
        _lib.lib()  # raises DeviceUnavailable without the library or a GPU
        dev = _device(device)
        hit = self._dev.get(dev.index)
        if hit is not None:
            return hit
        L = _lib.lib()
        with torch.cuda.device(dev):
            pts = torch.from_numpy(np.array(self.points)).to(dev)
            rec = torch.empty((_lib.record_rows(self.n), self.stride), dtype=torch.float64,
                              device=dev)
            sqmax = torch.zeros(1, dtype=torch.float64, device=dev)
            _lib.check(L.vr_pack_generators(_lib.ptr(pts), self.n, self.dim, _lib.ptr(rec),
                                            _lib.ptr(sqmax), _lib.stream_handle()),
                       "vr_pack_generators")
            entry = (rec, float(sqmax.item()))
        self._dev[dev.index] = entry
        return entry

    @property
    def fast_paths(self):
        """The fp32 screens and the kd-pruned kernels exist for d <= 8."""
        return self.dim <= FAST_MAX_DIM

    def screen32(self, device=None):
        """Centred fp32 copy of the records for the fp32 screen (built once);
        None for d > 8 (fp64 screen only)."""
        if not self.fast_paths:
            return None
        dev = _device(device)
        hit = self._s32.get(dev.index)
        if hit is None:
            rec, _ = self.device_records(dev)
            hit = Screen32(rec, self.n, self.dim)
            self._s32[dev.index] = hit
        return hit

    def prune_index(self, device=None):
        """kd-ordered records + tile / block bounding boxes for the pruned
        RayCast (include/voronray_b200.h vr_prune_index); built once per
        device on the GPU."""
        if not self.fast_paths:
            raise ValueError(f"the kd-pruned kernels cover d <= {FAST_MAX_DIM}; d={self.dim} "
                             "uses the exhaustive fp64 scan")
        dev = _device(device)
        hit = self._prune.get(dev.index)
        if hit is None:
            rec, _ = self.device_records(dev)
            hit = PruneIndex(rec, self.n, self.dim, self.screen32(dev).center)
            self._prune[dev.index] = hit
        return hit

    # -- filtered nearest neighbour (core.py:62-142) -------------------------
    def _skip_mask(self, skip):
        if skip is None:
            return None
        if callable(skip):
            return np.fromiter((bool(skip(i)) for i in range(self.n)), dtype=bool, count=self.n)
        return np.asarray(skip, dtype=bool)

    def _nearest_dev(self, q, skip):
        rec, _ = self.device_records()
        dev = rec.device
        L = _lib.lib()
        qd = torch.as_tensor(np.asarray(q, dtype=float).reshape(-1, self.dim), device=dev)
        mask = self._skip_mask(skip)
        md = None if mask is None else torch.as_tensor(mask.astype(np.uint8), device=dev)
        nq = qd.shape[0]
        idx = torch.empty(nq, dtype=torch.int32, device=dev)
        d1 = torch.empty(nq, dtype=torch.float64, device=dev)
        d2 = torch.empty(nq, dtype=torch.float64, device=dev)
        _lib.check(L.vr_nearest_batch(_lib.ptr(rec), self.n, self.dim, _lib.ptr(qd), nq,
                                      _lib.ptr(md), _lib.ptr(idx), _lib.ptr(d1), _lib.ptr(d2),
                                      _lib.stream_handle()), "vr_nearest_batch")
        return idx.cpu().numpy(), d1.cpu().numpy(), d2.cpu().numpy()

    def nearest(self, q, skip=None):
        """``(index, distance)`` of the nearest non-skipped point, or None."""
        idx, d1, _ = self._nearest_dev(q, skip)
        if idx[0] < 0:
            return None
        return int(idx[0]), float(d1[0])

    def nearest2(self, q, skip=None):
        """``((i, dist_i), dist_second)`` or None (core.py:105-142)."""
        idx, d1, d2 = self._nearest_dev(q, skip)
        if idx[0] < 0:
            return None
        return (int(idx[0]), float(d1[0])), float(d2[0])


PRUNE_TILE = 64  # VR_PRUNE_TILE of the library


class _Screen32Struct(ctypes.Structure):
    _fields_ = [("rec", ctypes.c_void_p), ("center", ctypes.c_double * 8),
                ("sqmax", ctypes.c_double), ("bound", ctypes.c_double),
                ("rec_pairs", ctypes.c_void_p)]


def screen_stats(rec, n, d, center=None):
    """(centre (d,) device fp64, sqmax, bound) of the fp32 screening frame of
    n packed records (vr_screen32_stats): the bounding-box midpoint unless
    `center` (device tensor) is given; one host read-back."""
    L = _lib.lib()
    stats = torch.empty(32, dtype=torch.float64, device=rec.device)
    _lib.check(L.vr_screen32_stats(_lib.ptr(rec), int(n), d, _lib.ptr(center), _lib.ptr(stats),
                                   _lib.stream_handle()), "vr_screen32_stats")
    host = stats[:10].cpu().numpy()
    return stats[:d].clone(), float(host[8]), float(host[9]), host[:d].tolist()


class Screen32:
    """Centred fp32 copy of a record array (include/voronray_b200.h vr_screen32)."""

    def __init__(self, rec, n, d, center=None):
        L = _lib.lib()
        dev = rec.device
        self.center, self.sqmax, self.bound, c_host = screen_stats(rec, n, d, center)
        s32 = (d + 4) & ~3
        self.rec = torch.empty((rec.shape[0], s32), dtype=torch.float32, device=dev)
        _lib.check(L.vr_pack_records32(_lib.ptr(rec), rec.shape[0], d, _lib.ptr(self.center),
                                       _lib.ptr(self.rec), _lib.stream_handle()),
                   "vr_pack_records32")
        rows = rec.shape[0]
        self.rec_pairs = torch.empty((rows // 2, (2 * d + 5) & ~3), dtype=torch.float32, device=dev)
        _lib.check(L.vr_pack_records32_pairs(_lib.ptr(self.rec), rows, d, _lib.ptr(self.rec_pairs),
                                             _lib.stream_handle()), "vr_pack_records32_pairs")
        c = [0.0] * 8
        c[:d] = c_host
        self.struct = _Screen32Struct(self.rec.data_ptr(), (ctypes.c_double * 8)(*c), self.sqmax,
                                      self.bound, self.rec_pairs.data_ptr())


class _PruneStruct(ctypes.Structure):
    _fields_ = [("rec", ctypes.c_void_p), ("rec32", ctypes.c_void_p), ("perm", ctypes.c_void_p),
                ("inv_perm", ctypes.c_void_p), ("tile_box", ctypes.c_void_p),
                ("tile_box32", ctypes.c_void_p), ("node_box", ctypes.c_void_p),
                ("node_box32", ctypes.c_void_p), ("node_range", ctypes.c_void_p),
                ("n", ctypes.c_int64), ("wide_box32", ctypes.c_void_p),
                ("wide_levels", ctypes.c_int32), ("wide_off", ctypes.c_int64 * 8),
                ("wide_cnt", ctypes.c_int64 * 8), ("recB", ctypes.c_void_p),
                ("rec32rows", ctypes.c_void_p), ("node_cb32", ctypes.c_void_p),
                ("recU", ctypes.c_void_p)]


class _PruneLayout(ctypes.Structure):
    _fields_ = [("arena_bytes", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("n_tiles", ctypes.c_int64), ("n_nodes", ctypes.c_int64),
                ("wide_levels", ctypes.c_int32)]


VR_PRUNE_MMA = 1
VR_PRUNE_UMMA = 2
MMA_MIN_D = int(os.environ.get("VR_MMA_MIN_D", "5"))  # tensor-core screen from this d


class PruneIndex:
    """One vr_prune_index, built natively (vr_build_prune_index) into a single
    device arena: kd-ordered records, perm / inv_perm, tile / node / 32-ary
    boxes and the fp32 / tensor-core screening copies.  The spatial index the
    reference builds in NodeSet.__init__ (core.py:52-57).  Tensor views of the
    arena are exposed for tests and tools."""

    def __init__(self, rec, n, d, center, workspace=None):
        L = _lib.lib()
        dev = rec.device
        # tensor-core screen operands from d = MMA_MIN_D: mma.sync fragments
        # (recB) and the canonical tcgen05 layout (recU); VR_MMA=0 disables
        flags = (VR_PRUNE_MMA | VR_PRUNE_UMMA) if (d >= MMA_MIN_D and
                                                   os.environ.get("VR_MMA", "2") != "0") else 0
        lay = _PruneLayout()
        _lib.check(L.vr_prune_index_layout(int(n), d, flags, ctypes.byref(lay)),
                   "vr_prune_index_layout")
        self.arena = torch.empty(int(lay.arena_bytes), dtype=torch.uint8, device=dev)
        if workspace is not None:
            ws = workspace.get("prune_build", (int(lay.workspace_bytes),), torch.uint8, dev)
        else:
            ws = torch.empty(int(lay.workspace_bytes), dtype=torch.uint8, device=dev)
        self.struct = _PruneStruct()
        _lib.check(L.vr_build_prune_index(_lib.ptr(rec), int(n), d, _lib.ptr(center), flags,
                                          _lib.ptr(self.arena), int(lay.arena_bytes), _lib.ptr(ws),
                                          int(lay.workspace_bytes), ctypes.byref(self.struct),
                                          _lib.stream_handle()), "vr_build_prune_index")
        del ws  # stream-ordered: the caching allocator reuses it after the build
        self.n, self.d, self.rows = int(n), d, _lib.record_rows(n)
        self.n_tiles, self.n_nodes = int(lay.n_tiles), int(lay.n_nodes)
        base = self.arena.data_ptr()
        st = self.struct

        def view(ptr, shape, dtype):
            if not ptr:
                return None
            esz = torch.empty(0, dtype=dtype).element_size()
            cnt = 1
            for x in shape:
                cnt *= int(x)
            off = int(ptr) - base
            return self.arena[off:off + cnt * esz].view(dtype).view(*shape)

        b32 = (2 * d + 3) & ~3
        ks = (d + 2 + 7) // 8
        self.rec = view(st.rec, (self.rows, (d + 2) & ~1), torch.float64)
        self.rec32rows = view(st.rec32rows, (self.rows, (d + 4) & ~3), torch.float32)
        self.rec32p = view(st.rec32, (self.rows // 2, (2 * d + 5) & ~3), torch.float32)
        self.perm = view(st.perm, (self.n,), torch.int32)
        self.inv_perm = view(st.inv_perm, (self.n,), torch.int32)
        self.tile_box = view(st.tile_box, (self.n_tiles, 2 * d), torch.float64)
        self.tile_box32 = view(st.tile_box32, (self.n_tiles, b32), torch.float32)
        self.node_box = view(st.node_box, (self.n_nodes, 2 * d), torch.float64)
        self.node_box32 = view(st.node_box32, (self.n_nodes, b32), torch.float32)
        self.node_cb32 = view(st.node_cb32, (self.n_nodes, b32), torch.float32)
        self.node_range = view(st.node_range, (self.n_nodes, 2), torch.int32)
        self.wide_cnt = [int(st.wide_cnt[i]) for i in range(st.wide_levels)]
        self.wide_off = [int(st.wide_off[i]) for i in range(st.wide_levels)]
        self.wide_box32 = view(st.wide_box32, (sum(self.wide_cnt), b32), torch.float32)
        self.recB = view(st.recB, (self.rows, 8 * ks), torch.float32)
        self.recU = view(st.recU, (self.rows, 8 * ks), torch.float32)


def build_node_set(points, backend="auto"):
    """Validate raw coordinates and build a :class:`NodeSet` (core.py:145-169)."""
    rows = [np.asarray(p, dtype=float) for p in points]
    if not rows:
        raise DimensionMismatch("empty point set")
    d = rows[0].shape[-1] if rows[0].ndim else 0
    for p in rows:
        if p.ndim != 1 or p.shape[0] != d:
            raise DimensionMismatch("all points must share one dimension")
    if d < 2:
        raise DimensionMismatch("dimension must be at least 2")
    if len(rows) < d + 1:
        raise DimensionMismatch(f"need at least d+1={d + 1} points, got {len(rows)}")
    arr = np.vstack(rows)
    # exact duplicates: identical byte rows (core.py:163-168), vectorised
    _, first = np.unique(arr.view(np.dtype((np.void, arr.dtype.itemsize * d))).ravel(),
                         return_index=True)
    if first.size != arr.shape[0]:
        dup_mask = np.ones(arr.shape[0], dtype=bool)
        dup_mask[first] = False
        raise DuplicatePoint(f"duplicate coordinates {arr[np.argmax(dup_mask)].tolist()}")
    return NodeSet(arr, backend=backend)


def nearest_neighbor(ns: NodeSet, q, skip=None):
    """Nearest node to ``q`` among non-skipped indices (core.py:172-181)."""
    q = np.asarray(q, dtype=float)
    if q.shape != (ns.dim,):
        raise DimensionMismatch(f"query must have length {ns.dim}")
    return ns.nearest(q, skip)


@dataclass(frozen=True)
class VertexRecord:
    """A Voronoi vertex: sorted generator indices plus its coordinate."""

    sigma: tuple
    r: np.ndarray


@dataclass(frozen=True)
class BoundaryRay:
    """An unbounded edge anchored at vertex ``sigma`` with direction ``u``."""

    sigma: tuple
    u: np.ndarray


def edge_keys(sigma):
    """All d-subsets of the sorted (d+1)-tuple ``sigma`` (core.py:200-202)."""
    return [sigma[:k] + sigma[k + 1:] for k in range(len(sigma))]


class Mesh:
    """Traversal output with array storage and lazy reference-style views.

    Constructed either like the reference dataclass
    ``Mesh(nodes, vertices, edge_counts, boundary)`` (core.py:205-221) or from
    device-produced arrays via :meth:`from_arrays`.
    """

    def __init__(self, nodes, vertices=None, edge_counts=None, boundary=None):
        self.nodes = nodes
        self._vertices = vertices
        self._edge_counts = edge_counts
        self._boundary = boundary
        self._arr = None
        self._dev = None
        self._cell_csr = None
        self._neighbors = {}
        self._unbounded = None
        self._unbounded_faces = None

    # -- array form -------------------------------------------------------
    @classmethod
    def from_arrays(cls, nodes, sigma, r, edge_key, edge_count, boundary_sigma, boundary_u):
        m = cls(nodes)
        m._arr = dict(sigma=np.ascontiguousarray(sigma, dtype=np.int32),
                      r=np.ascontiguousarray(r, dtype=np.float64),
                      edge_key=np.ascontiguousarray(edge_key, dtype=np.int32),
                      edge_count=np.ascontiguousarray(edge_count, dtype=np.int32),
                      boundary_sigma=np.ascontiguousarray(boundary_sigma, dtype=np.int32),
                      boundary_u=np.ascontiguousarray(boundary_u, dtype=np.float64))
        return m

    @classmethod
    def from_device(cls, nodes, sigma, r, edge_key, edge_count, boundary_sigma, boundary_u):
        """Mesh over device tensors (traversal output), kept resident in HBM:
        the host arrays (and the lexicographic edge order) are produced on
        first access, so a traversal whose result is consumed on the device
        (or only counted) never pays for the device -> host copy."""
        m = cls(nodes)
        m._dev = dict(sigma=sigma, r=r, edge_key=edge_key, edge_count=edge_count,
                      boundary_sigma=boundary_sigma, boundary_u=boundary_u)
        return m

    def device_arrays(self):
        """The device tensors of a traversal mesh (edges in hash order), or None."""
        return self._dev

    def _materialize(self):
        import torch
        dv = self._dev
        ek, ec = dv["edge_key"], dv["edge_count"]
        if ek.shape[0]:  # the reference's sorted(edge_counts) order (vr_lex_order)
            order = lex_order(ek)
            ek, ec = ek.index_select(0, order), ec.index_select(0, order)

        def host(t, dtype):
            t = t.contiguous()
            if t.is_cuda and t.numel():
                buf = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                buf.copy_(t)
                t = buf
            return np.ascontiguousarray(t.cpu().numpy(), dtype=dtype)

        self._arr = dict(sigma=host(dv["sigma"], np.int32), r=host(dv["r"], np.float64),
                         edge_key=host(ek, np.int32), edge_count=host(ec, np.int32),
                         boundary_sigma=host(dv["boundary_sigma"], np.int32),
                         boundary_u=host(dv["boundary_u"], np.float64))

    def arrays(self):
        """sigma (V, d+1) int32, r (V, d), edge_key (E, d), edge_count (E,),
        boundary_sigma (B, d+1), boundary_u (B, d)."""
        if self._arr is None and self._dev is not None:
            self._materialize()
        if self._arr is None:
            d = self.nodes.dim
            verts = list(self._vertices.values()) if self._vertices else []
            sig = np.array([v.sigma for v in verts], dtype=np.int32).reshape(-1, d + 1)
            r = np.array([v.r for v in verts], dtype=np.float64).reshape(-1, d)
            ek = np.array(list(self._edge_counts.keys()) if self._edge_counts else [],
                          dtype=np.int32).reshape(-1, d)
            ec = np.array(list(self._edge_counts.values()) if self._edge_counts else [],
                          dtype=np.int32)
            bl = self._boundary or []
            bs = np.array([b.sigma for b in bl], dtype=np.int32).reshape(-1, d + 1)
            bu = np.array([b.u for b in bl], dtype=np.float64).reshape(-1, d)
            self._arr = dict(sigma=sig, r=r, edge_key=ek, edge_count=ec,
                             boundary_sigma=bs, boundary_u=bu)
        return self._arr

    @property
    def n_vertices(self):
        if self._arr is None and self._dev is not None:
            return int(self._dev["sigma"].shape[0])
        return self.arrays()["sigma"].shape[0]

    @property
    def vertices(self):
        if self._vertices is None:
            a = self.arrays()
            self._vertices = {tuple(int(x) for x in s): VertexRecord(tuple(int(x) for x in s), r)
                              for s, r in zip(a["sigma"], a["r"])}
        return self._vertices

    @vertices.setter
    def vertices(self, value):
        self._vertices = value
        self._arr = None
        self._dev = None

    @property
    def edge_counts(self):
        if self._edge_counts is None:
            a = self.arrays()
            self._edge_counts = {tuple(int(x) for x in k): int(c)
                                 for k, c in zip(a["edge_key"], a["edge_count"])}
        return self._edge_counts

    @property
    def boundary(self):
        if self._boundary is None:
            a = self.arrays()
            self._boundary = [BoundaryRay(tuple(int(x) for x in s), u)
                              for s, u in zip(a["boundary_sigma"], a["boundary_u"])]
        return self._boundary

    def contains(self, sigma):
        """Membership of sorted sigma rows in the vertex set (the reference's
        ``sigma in mesh.vertices``, core.py:205-221), vectorised: bool array.
        A device-resident traversal mesh is searched on the device (64-bit
        row hashes, sorted once, exact row comparison of the hash matches),
        so nothing is copied to the host."""
        d1 = self.nodes.dim + 1
        q = np.ascontiguousarray(sigma, dtype=np.int32).reshape(-1, d1)
        if self._dev is not None and self._arr is None:
            S = self._dev["sigma"]
            if S.shape[0] == 0 or q.shape[0] == 0:
                return np.zeros(q.shape[0], dtype=bool)
            if getattr(self, "_hash_index", None) is None:
                h = _row_hash(S)
                hs, order = torch.sort(h)
                self._hash_index = (hs, order)
            hs, order = self._hash_index
            qd = torch.from_numpy(q).to(S.device)
            qh = _row_hash(qd)
            pos = torch.searchsorted(hs, qh)
            found = torch.zeros(q.shape[0], dtype=torch.bool, device=S.device)
            last = S.shape[0] - 1
            for k in range(4):  # equal hashes are adjacent; 4 covers any real collision
                pk = (pos + k).clamp(max=last)
                found |= (hs[pk] == qh) & (S[order[pk]] == qd).all(1)
            return found.cpu().numpy()
        a = self.arrays()["sigma"]
        have = {tuple(r) for r in a.tolist()}
        return np.array([tuple(r) in have for r in q.tolist()], dtype=bool)

    # -- cell maps (core.py:223-276) ---------------------------------------
    def _csr(self):
        if self._cell_csr is None:
            sig = self.arrays()["sigma"] if self._vertices is None else None
            if sig is None:
                keys = list(self._vertices.keys())
                sig = np.array(keys, dtype=np.int32).reshape(-1, self.nodes.dim + 1)
                self._vlist = [self._vertices[k] for k in keys]
            else:
                self._vlist = None
            flat = sig.ravel()
            vid = np.repeat(np.arange(sig.shape[0]), sig.shape[1])
            order = np.argsort(flat, kind="stable")
            counts = np.bincount(flat, minlength=self.nodes.n)
            off = np.zeros(self.nodes.n + 1, dtype=np.int64)
            np.cumsum(counts, out=off[1:])
            self._cell_csr = (off, vid[order], sig)
        return self._cell_csr

    def _vertex(self, v):
        if getattr(self, "_vlist", None) is not None:
            return self._vlist[v]
        a = self.arrays()
        s = tuple(int(x) for x in a["sigma"][v])
        return self.vertices[s]

    def cell_vertices(self, i):
        off, vids, _ = self._csr()
        if i < 0 or i >= self.nodes.n:
            return []
        return [self._vertex(int(v)) for v in vids[off[i]:off[i + 1]]]

    def neighbors(self, i):
        hit = self._neighbors.get(i)
        if hit is None:
            off, vids, sig = self._csr()
            if 0 <= i < self.nodes.n and off[i + 1] > off[i]:
                s = np.unique(sig[vids[off[i]:off[i + 1]]])
                hit = tuple(int(x) for x in s if x != i)
            else:
                hit = ()
            self._neighbors[i] = hit
        return hit

    def unbounded_cells(self):
        if self._unbounded is None:
            out = set()
            for eta, c in self.edge_counts.items():
                if c == 1:
                    out.update(eta)
            self._unbounded = frozenset(out)
        return self._unbounded

    def bounded_cells(self):
        unb = self.unbounded_cells()
        off, _, _ = self._csr()
        return [i for i in range(self.nodes.n) if i not in unb and off[i + 1] > off[i]]

    def face_vertices(self, i, j):
        return [v for v in self.cell_vertices(i) if j in v.sigma]

    def face_is_unbounded(self, i, j):
        if self._unbounded_faces is None:
            pairs = set()
            for eta, c in self.edge_counts.items():
                if c == 1:
                    pairs.update(combinations(eta, 2))
            self._unbounded_faces = frozenset(pairs)
        key = (i, j) if i < j else (j, i)
        return key in self._unbounded_faces


def lex_order(rows):
    """Stable lexicographic row order of an int32 device tensor (vr_lex_order)."""
    rows = rows.to(torch.int32).contiguous()
    n, k = rows.shape
    L = _lib.lib()
    nb = ctypes.c_int64(0)
    _lib.check(L.vr_lex_order(None, n, k, None, None, ctypes.byref(nb), None), "vr_lex_order")
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=rows.device)
    order = torch.empty(n, dtype=torch.int32, device=rows.device)
    _lib.check(L.vr_lex_order(_lib.ptr(rows), n, k, _lib.ptr(order), _lib.ptr(ws),
                              ctypes.byref(nb), _lib.stream_handle()), "vr_lex_order")
    return order.long()


def edge_incidence(ns, sigma):
    """(distinct edge keys (E, d) lexicographic, incidence counts (E,)) of the
    sigma rows, on the device (vr_edge_incidence)."""
    rec, _ = ns.device_records()
    dev = rec.device
    d = ns.dim
    sig = (sigma if isinstance(sigma, torch.Tensor) else torch.as_tensor(
        np.ascontiguousarray(sigma, dtype=np.int32))).to(device=dev, dtype=torch.int32)
    sig = sig.reshape(-1, d + 1).contiguous()
    nv = sig.shape[0]
    L = _lib.lib()
    nb = ctypes.c_int64(0)
    nu = ctypes.c_int64(0)
    _lib.check(L.vr_edge_incidence(None, nv, d, None, None, None, None, ctypes.byref(nb), None),
               "vr_edge_incidence (size)")
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=dev)
    keys = torch.empty((max(nv * (d + 1), 1), d), dtype=torch.int32, device=dev)
    cnt = torch.empty(max(nv * (d + 1), 1), dtype=torch.int32, device=dev)
    _lib.check(L.vr_edge_incidence(_lib.ptr(sig), nv, d, _lib.ptr(keys), _lib.ptr(cnt),
                                   ctypes.byref(nu), _lib.ptr(ws), ctypes.byref(nb),
                                   _lib.stream_handle()), "vr_edge_incidence")
    return keys[:nu.value], cnt[:nu.value]


def _row_hash(rows):
    """64-bit polynomial hash of int32 rows (device tensor), wrapping."""
    h = torch.zeros(rows.shape[0], dtype=torch.int64, device=rows.device)
    for k in range(rows.shape[1]):
        h = h * 1000003 + rows[:, k].to(torch.int64)
        h = h ^ (h >> 29)
    return h


def verify_vertices_device(ns: NodeSet, sigma, r, tol: float = TOL_VERTEX):
    """verify_vertex (core.py:279-296) for device tensors sigma (V, d+1) /
    r (V, d): equidistance and the incircle scan against all N generators
    (vr_verify_vertices); a device bool tensor."""
    rec, _ = ns.device_records()
    dev = rec.device
    sd = sigma.to(device=dev, dtype=torch.int32).reshape(-1, ns.dim + 1).contiguous()
    rd = r.to(device=dev, dtype=torch.float64).reshape(-1, ns.dim).contiguous()
    ok = torch.empty(sd.shape[0], dtype=torch.uint8, device=dev)
    if sd.shape[0]:
        _lib.check(_lib.lib().vr_verify_vertices(_lib.ptr(rec), ns.n, ns.dim, _lib.ptr(sd),
                                                 _lib.ptr(rd), sd.shape[0], float(tol),
                                                 _lib.ptr(ok), _lib.stream_handle()),
                   "vr_verify_vertices")
    return ok.bool()


def verify_vertices(ns: NodeSet, sigma, r, tol: float = TOL_VERTEX):
    """Batched verify_vertex on the GPU: bool array, one per vertex."""
    sigma = np.ascontiguousarray(sigma, dtype=np.int32).reshape(-1, ns.dim + 1)
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1, ns.dim)
    if sigma.shape[0] == 0:
        return np.zeros(0, dtype=bool)
    ok = verify_vertices_device(ns, torch.from_numpy(sigma), torch.from_numpy(r), tol)
    return ok.cpu().numpy()


def verify_vertex(mesh: Mesh, v: VertexRecord, tol: float = TOL_VERTEX) -> bool:
    """Equidistance + incircle invariants of one vertex (core.py:279-296)."""
    ns = mesh.nodes
    sig = list(v.sigma)
    if len(sig) != ns.dim + 1 or len(set(sig)) != len(sig):
        return False
    return bool(verify_vertices(ns, np.array([sig]), np.asarray(v.r)[None], tol)[0])
