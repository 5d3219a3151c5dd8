"""Incircle RayCast on the B200 (drop-in for voronray.raycast).

``raycast_batch`` is the real entry point: one fused sm_100a kernel over
rays x generators (csrc/raycast_core.cuh) computes, for every ray, the
converged answer of the reference's incircle probe loop
(pkg/src/voronray/raycast.py:154-224) -- the valid generator with the
smallest crossing parameter -- plus the exact re-check pass for rays whose
decision lies inside the degeneracy / rounding band.  ``raycast_incircle``
keeps the reference signature, return type and exceptions on top of it.

The small helpers (``project_t``, ``initial_heuristic``, ``search_direction``,
``_vertex_directions``, Gram-Schmidt) are host-side scalar geometry with the
reference semantics (raycast.py:49-82, 295-378); they are not on the hot path.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import NodeSet
from .errors import DegenerateConfiguration, ParallelGenerator

PARALLEL_TOL = 1e-14
RANK_TOL = 1e-10

RAY_OK, RAY_ESCAPED, RAY_RECHECK, RAY_DEGENERATE = 0, 1, 2, 3


@dataclass(slots=True)
class RayQuery:
    """Edge/face ray: generator indices ``eta``, anchor ``r``, direction ``u``."""

    eta: tuple
    r: np.ndarray
    u: np.ndarray


@dataclass
class RaycastStats:
    """Counters (raycast.py:40-46).  On the GPU one fused candidate scan
    replaces the whole probe loop, so each raycast counts one ``nn_calls``
    and one ``iterations``."""

    nn_calls: int = 0
    iterations: int = 0
    raycasts: int = 0

    def add(self, n):
        self.raycasts += n
        self.nn_calls += n
        self.iterations += n


def project_t(r, u, x0, x):
    """Ray parameter of the point equidistant to ``x0`` and ``x`` (raycast.py:49-65)."""
    dx = x - x0
    denom = float(np.dot(u, dx))
    scale = float(np.linalg.norm(dx))
    if abs(denom) < PARALLEL_TOL * scale:
        raise ParallelGenerator("candidate generator lies in the search hyperplane")
    a = r - x
    b = r - x0
    return (float(a @ a) - float(b @ b)) / (2.0 * denom)


def initial_heuristic(q: RayQuery, x):
    """Regular-simplex warm start (raycast.py:68-82).  Result-neutral: the GPU
    kernel scans every candidate, so it is provided for API parity only."""
    k = len(q.eta)
    if k < 2:
        raise ValueError("heuristic needs at least two known generators")
    rp = q.r + q.u * float(q.u @ (x - q.r))
    rx = rp - x
    radius = math.sqrt(float(rx @ rx))
    return rp + q.u * (radius / math.sqrt((k - 1) * (k + 1)))


def _as_dev(a, dev, dtype):
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev)


class RaycastBatch:
    """Device-resident results of one batched RayCast.

    idx (int32, -1 = escaped), t (fp64), rp (fp64 (n, d) or None),
    flag (uint8: 0 ok, 1 escaped, 3 degenerate).
    """

    def __init__(self, idx, t, rp, flag):
        self.idx, self.t, self.rp, self.flag = idx, t, rp, flag

    def to_host(self):
        h = _lib.to_host
        return (h(self.idx), h(self.t), None if self.rp is None else h(self.rp), h(self.flag))


class Workspace:
    """Reusable device buffers for repeated batches of the same size."""

    def __init__(self):
        self._bufs = {}

    def get(self, name, shape, dtype, dev):
        t = self._bufs.get(name)
        n = 1
        for s in shape:  # (np.prod costs ~5 us; the traversal calls this ~15x per level)
            n *= int(s)
        if t is None or t.numel() < n or t.dtype != dtype or t.device != dev:
            t = torch.empty(max(n, 1), dtype=dtype, device=dev)
            self._bufs[name] = t
        return t[:n].view(shape)


def candidate_records(ns: NodeSet, candidates, dev, screen="fp64"):
    """Packed records of a candidate subset (raycast.py:100-102); with
    screen="fp32" also the matching centred fp32 rows (vr_screen32 struct)."""
    rec, _ = ns.device_records(dev)
    cand = _as_dev(np.asarray(candidates, dtype=np.int64).ravel(), dev, torch.int64)
    m = cand.shape[0]
    crec = torch.zeros((_lib.record_rows(m), rec.shape[1]), dtype=rec.dtype, device=dev)
    crec[:, ns.dim] = float("inf")  # sentinel rows (include/voronray_b200.h)
    crec[:m] = rec.index_select(0, cand)
    s32 = None
    if screen == "fp32" and ns.fast_paths:
        from .core import Screen32
        s32 = Screen32(crec, m, ns.dim, center=ns.screen32(dev).center)
    return cand.to(torch.int32).contiguous(), crec, s32


def direction_bucket(u):
    """Coarse direction class of unit vectors: the signed index of the
    largest and of the second-largest |component| (< 256 classes for d <= 8)."""
    d = u.shape[1]
    a = u.abs()
    i1 = a.argmax(1)
    s1 = (u.gather(1, i1[:, None])[:, 0] > 0).to(torch.int64)
    a2 = a.scatter(1, i1[:, None], -1.0)
    i2 = a2.argmax(1)
    s2 = (u.gather(1, i2[:, None])[:, 0] > 0).to(torch.int64)
    return (i1 * 2 + s1) * (2 * d) + (i2 * 2 + s2)


def ray_keys(u, eta=None, inv_perm=None, rays_per_cell=1):
    """Processing-order keys on the device (vr_ray_keys): base * 256 +
    direction_bucket(u), base = inv_perm[eta[:, 0]] or, without eta,
    k // rays_per_cell."""
    n, d = u.shape
    keys = torch.empty(n, dtype=torch.int64, device=u.device)
    L = _lib.lib()
    if eta is not None:
        eta = eta.view(n, -1)
        _lib.check(L.vr_ray_keys(_lib.ptr(inv_perm), _lib.ptr(eta), eta.shape[1], 1,
                                 _lib.ptr(u), n, d, _lib.ptr(keys), _lib.stream_handle()),
                   "vr_ray_keys")
    else:
        _lib.check(L.vr_ray_keys(None, None, 0, int(rays_per_cell), _lib.ptr(u), n, d,
                                 _lib.ptr(keys), _lib.stream_handle()), "vr_ray_keys")
    return keys


def ray_order(u, eta=None, inv_perm=None, rays_per_cell=1, n_base=None, workspace=None,
              stream=None):
    """Processing order of a ray batch for the pruned kernels (vr_ray_order:
    the vr_ray_keys keys, 32-bit when they fit, sorted by the library's own
    stable radix sort): int32 device tensor, slot -> ray id.  `n_base` is
    the range of the key base (the generator count, or the cell count when
    eta is None); buffers come from `workspace` when given."""
    n, d = u.shape
    dev = u.device
    L = _lib.lib()
    nbytes = ctypes.c_int64(0)
    _lib.check(L.vr_ray_order(None, None, d, 1, None, n, d, int(n_base), None, None,
                              ctypes.byref(nbytes), None), "vr_ray_order (size)")
    if workspace is not None:
        tmp = workspace.get("order_tmp", (max(1, nbytes.value),), torch.uint8, dev)
        order = workspace.get("order", (n,), torch.int32, dev)
    else:
        tmp = torch.empty(max(1, nbytes.value), dtype=torch.uint8, device=dev)
        order = torch.empty(n, dtype=torch.int32, device=dev)
    if eta is not None:
        eta = eta.view(n, -1)
        _lib.check(L.vr_ray_order(_lib.ptr(inv_perm), _lib.ptr(eta), eta.shape[1], 1, _lib.ptr(u),
                                  n, d, int(n_base), _lib.ptr(order), _lib.ptr(tmp),
                                  ctypes.byref(nbytes), _lib.stream_handle(stream)),
                   "vr_ray_order")
    else:
        _lib.check(L.vr_ray_order(None, None, 0, int(rays_per_cell), _lib.ptr(u), n, d,
                                  int(n_base), _lib.ptr(order), _lib.ptr(tmp),
                                  ctypes.byref(nbytes), _lib.stream_handle(stream)),
                   "vr_ray_order")
    return order


def coherent_order(ix, eta, u, workspace=None, stream=None):
    """Processing order for the pruned kernel: rays sorted by the kd position
    of their reference generator (eta[:, 0]), then by direction class, so
    that the 32 rays of a warp start close together and (within one
    generator) point the same way -- the warp-wide union of their spheres
    stays small.  (Scheduling the longest, near-hull warps first was
    measured slower: it breaks the locality of consecutive warps.)"""
    return ray_order(u.contiguous(), eta.to(torch.int32).contiguous(), ix.inv_perm,
                     n_base=ix.n, workspace=workspace, stream=stream)


def _screen(ns, dev, screen):
    if screen not in ("fp32", "fp64"):
        raise ValueError(f"unknown screen {screen!r}")
    return ns.screen32(dev) if screen == "fp32" else None  # None for d > 8: fp64


PRUNE_MIN_GENERATORS = 256  # below: one exhaustive scan is as fast (config 1 uses pruned: 19 -> 17 ms)


def _use_pruned(ns, candidates, mode):
    if mode not in ("auto", "pruned", "exhaustive"):
        raise ValueError(f"unknown mode {mode!r}")
    if candidates is not None or mode == "exhaustive" or not ns.fast_paths:
        return False
    return mode == "pruned" or ns.n >= PRUNE_MIN_GENERATORS


def raycast_batch(ns: NodeSet, x, u, eta, candidates=None, want_rp=True, stats=None,
                  workspace=None, out=None, stream=None, events=None,
                  mode="auto", work=None, screen="fp32") -> RaycastBatch:
    """Batched incircle RayCast on the current CUDA device.

    Args:
        ns: node set.
        x: (n, d) ray origins, equidistant to their eta generators.
        u: (n, d) unit directions.
        eta: (n, k) generator indices per ray (1 <= k <= d); eta[:, 0] is the
            reference generator x0 of the crossing formula (raycast.py:182).
        candidates: optional index subset restricting the search.
        want_rp: also return the new vertex coordinates x + t u.
        out: optional dict of preallocated output tensors (idx, t, rp, flag).
        events: optional three CUDA events recorded before the fused kernel,
            between it and the re-check pass, and after (kernel timing).
        mode: "exhaustive" scans every generator (TMA-staged tiles);
            "pruned" skips kd tiles with a certificate (identical results);
            "auto" prunes when N >= PRUNE_MIN_GENERATORS and no candidate subset is given.
        work: optional zeroed int64 device tensor of >= 16 entries (see
            VR_WORK_COUNTERS in the header); [0] accumulates the pairs the
            pruned kernel screened (roofline accounting).
        screen: "fp32" screens pairs in fp32 (centred frame, rigorous bound)
            and re-checks survivors in fp64; "fp64" screens in fp64.  The
            results are identical (tests/test_raycast_gpu.py).

    Stream-ordered; no host synchronisation.
    """
    rec, sqmax = ns.device_records()
    dev = rec.device
    L = _lib.lib()
    d = ns.dim
    xd = _as_dev(x, dev, torch.float64).view(-1, d)
    ud = _as_dev(u, dev, torch.float64).view(-1, d)
    n = xd.shape[0]
    ed = _as_dev(eta, dev, torch.int32)
    if ed.dim() == 1:
        ed = ed.view(n, -1) if n else ed.view(0, 1)
    k = ed.shape[1] if ed.dim() == 2 else 1
    if not 1 <= k <= d:
        raise ValueError(f"eta must hold between 1 and d={d} generators, got {k}")
    if ud.shape[0] != n or ed.shape[0] != n:
        raise ValueError("x, u and eta must describe the same number of rays")
    ws = workspace or Workspace()
    if out is None:
        out = {}
    idx = out.get("idx") if out.get("idx") is not None else torch.empty(n, dtype=torch.int32, device=dev)
    t = out.get("t") if out.get("t") is not None else torch.empty(n, dtype=torch.float64, device=dev)
    flag = out.get("flag") if out.get("flag") is not None else torch.empty(n, dtype=torch.uint8, device=dev)
    rp = None
    if want_rp:
        rp = out.get("rp") if out.get("rp") is not None else torch.empty((n, d), dtype=torch.float64, device=dev)
    if stats is not None:
        stats.add(n)
    if n == 0:
        return RaycastBatch(idx, t, rp, flag)
    cand = crec = None
    n_cand = 0
    s32 = _screen(ns, dev, screen)
    if candidates is not None:
        if len(np.asarray(candidates).ravel()) == 0:
            # reference _Probe with an empty candidate array: every probe is
            # all-invalid, so the ray escapes (raycast.py:100-102, 188-191)
            idx.fill_(-1)
            t.fill_(float("nan"))
            flag.fill_(RAY_ESCAPED)
            if rp is not None:
                rp.fill_(float("nan"))
            return RaycastBatch(idx, t, rp, flag)
        cand, crec, s32 = candidate_records(ns, candidates, dev, screen)
        n_cand = cand.shape[0]
    s32p = ctypes.byref(s32.struct) if s32 is not None else None
    rl = ws.get("recheck_list", (n,), torch.int32, dev)
    rc = ws.get("recheck_count", (1,), torch.int32, dev)
    sh = _lib.stream_handle(stream)
    pruned = _use_pruned(ns, candidates, mode)
    if work is not None and work.numel() < 16:
        raise ValueError("work must hold at least 16 counters (VR_WORK_COUNTERS)")
    if events is not None:
        events[0].record(stream)
    if pruned:
        ix = ns.prune_index(dev)
        order = coherent_order(ix, ed, ud, workspace=ws, stream=stream)
        _lib.check(L.vr_raycast_pruned(_lib.ptr(rec), ns.n, d, sqmax, s32p, ctypes.byref(ix.struct),
                                       _lib.ptr(xd), _lib.ptr(ud), _lib.ptr(ed), k, n,
                                       _lib.ptr(order), _lib.ptr(idx), _lib.ptr(t),
                                       _lib.ptr(rp), _lib.ptr(flag), _lib.ptr(rl), _lib.ptr(rc),
                                       _lib.ptr(work), sh), "vr_raycast_pruned")
    else:
        _lib.check(L.vr_raycast_batch(_lib.ptr(rec), ns.n, d, sqmax, s32p, _lib.ptr(crec),
                                      _lib.ptr(cand), n_cand, _lib.ptr(xd), _lib.ptr(ud),
                                      _lib.ptr(ed), k, n, _lib.ptr(idx), _lib.ptr(t),
                                      _lib.ptr(rp), _lib.ptr(flag), _lib.ptr(rl), _lib.ptr(rc),
                                      sh), "vr_raycast_batch")
    if events is not None:
        events[1].record(stream)
    _lib.check(L.vr_raycast_recheck(_lib.ptr(rec), ns.n, d, _lib.ptr(crec), _lib.ptr(cand),
                                    n_cand, _lib.ptr(xd), _lib.ptr(ud), _lib.ptr(ed), k,
                                    _lib.ptr(rl), _lib.ptr(rc), n, _lib.ptr(idx), _lib.ptr(t),
                                    _lib.ptr(rp), _lib.ptr(flag), sh), "vr_raycast_recheck")
    if events is not None:
        events[2].record(stream)
    return RaycastBatch(idx, t, rp, flag)


def raycast_incircle(ns: NodeSet, q: RayQuery, stats: RaycastStats = None,
                     heuristic: bool = True, candidates=None):
    """Exact first Voronoi object hit by the ray, or None if it escapes.

    Drop-in for raycast.py:154-224: returns ``(tuple(sorted(eta + (i,))), rp)``
    or ``None``; raises :class:`DegenerateConfiguration` when a foreign
    generator lies within the reference's 1e-10 band of the circumsphere.
    ``heuristic`` is result-neutral in the reference and ignored here.
    """
    if stats is None:
        stats = RaycastStats()
    eta = tuple(int(e) for e in q.eta)
    if candidates is None and 1 <= len(eta) <= ns.dim:
        i, f, rp = _single_ray(ns, q.r, q.u, eta, stats)
    else:
        res = raycast_batch(ns, np.asarray(q.r, dtype=float)[None],
                            np.asarray(q.u, dtype=float)[None], np.asarray([eta], dtype=np.int32),
                            candidates=candidates, stats=stats)
        idx, _, rpa, flag = res.to_host()
        i, f, rp = int(idx[0]), int(flag[0]), rpa[0]
    if f == RAY_ESCAPED:
        return None
    if f == RAY_DEGENERATE:
        raise DegenerateConfiguration(
            f"a foreign generator lies on the circumsphere of {(*eta, i)}")
    return tuple(sorted((*eta, i))), rp


class _SingleRay:
    """Reused buffers of the one-ray drop-in call (raycast_incircle): the
    inputs packed in one pinned host block and copied with one H2D, the
    outputs (rp, t, idx, flag) views of one device block read back with one
    D2H -- a call is the RayCast launches plus two copies and one sync, with
    no per-call allocations (the reference's loops, descent and the DFS, call
    it once per step)."""

    def __init__(self, ns, k):
        rec, _ = ns.device_records()
        self.dev, d = rec.device, ns.dim
        self.k = k
        self.nin = 16 * d + 4 * k
        self.nout = 8 * d + 16
        self.h_in = torch.empty(self.nin, dtype=torch.uint8, pin_memory=True)
        self.h_out = torch.empty(self.nout, dtype=torch.uint8, pin_memory=True)
        self.d_in = torch.empty(self.nin, dtype=torch.uint8, device=self.dev)
        self.d_out = torch.empty(self.nout, dtype=torch.uint8, device=self.dev)
        hi = self.h_in.numpy()
        self.hx = hi[:8 * d].view(np.float64)
        self.hu = hi[8 * d:16 * d].view(np.float64)
        self.he = hi[16 * d:].view(np.int32)
        self.x = self.d_in[:8 * d].view(torch.float64).view(1, d)
        self.u = self.d_in[8 * d:16 * d].view(torch.float64).view(1, d)
        self.eta = self.d_in[16 * d:].view(torch.int32).view(1, k)
        self.out = dict(rp=self.d_out[:8 * d].view(torch.float64).view(1, d),
                        t=self.d_out[8 * d:8 * d + 8].view(torch.float64),
                        idx=self.d_out[8 * d + 8:8 * d + 12].view(torch.int32),
                        flag=self.d_out[8 * d + 12:8 * d + 13])
        ho = self.h_out.numpy()
        self.h_rp = ho[:8 * d].view(np.float64)
        self.h_idx = ho[8 * d + 8:8 * d + 12].view(np.int32)
        self.h_flag = ho[8 * d + 12:8 * d + 13]
        self.ws = Workspace()


def _single_ray(ns, r, u, eta, stats):
    cache = ns.__dict__.setdefault("_single_ray_bufs", {})
    sb = cache.get(len(eta))
    if sb is None:
        sb = cache[len(eta)] = _SingleRay(ns, len(eta))
    sb.hx[:] = np.asarray(r, dtype=np.float64).ravel()
    sb.hu[:] = np.asarray(u, dtype=np.float64).ravel()
    sb.he[:] = eta
    sb.d_in.copy_(sb.h_in, non_blocking=True)
    raycast_batch(ns, sb.x, sb.u, sb.eta, out=sb.out, workspace=sb.ws, stats=stats)
    sb.h_out.copy_(sb.d_out, non_blocking=True)
    torch.cuda.current_stream(sb.dev).synchronize()
    return int(sb.h_idx[0]), int(sb.h_flag[0]), sb.h_rp.copy()


# --- host-side direction helpers (raycast.py:295-378) ----------------------

def _orthonormal_rows(diffs):
    """Modified Gram-Schmidt, two passes (raycast.py:295-308)."""
    out = []
    for row in np.atleast_2d(diffs) if len(diffs) else []:
        v = np.array(row, dtype=float)
        norm0 = math.sqrt(float(v @ v))
        for _ in range(2):
            for qv in out:
                v -= (qv @ v) * qv
        norm = math.sqrt(float(v @ v))
        if norm < RANK_TOL * max(norm0, 1.0):
            raise DegenerateConfiguration("generators are affinely dependent")
        out.append(v / norm)
    return out


def _project_out(w, basis):
    """Component of ``w`` orthogonal to orthonormal rows (raycast.py:311-317)."""
    v = np.array(w, dtype=float)
    for _ in range(2):
        for qv in basis:
            v -= (qv @ v) * qv
    return v


def _search_direction(pts, eta, missing):
    sub = pts[list(eta)]
    basis = _orthonormal_rows(sub[1:] - sub[0]) if len(eta) > 1 else []
    w = sub.sum(axis=0) * (1.0 / len(eta)) - pts[missing]
    v = _project_out(w, basis)
    norm = math.sqrt(float(v @ v))
    if norm < RANK_TOL * max(math.sqrt(float(w @ w)), 1.0):
        raise DegenerateConfiguration(f"generator {missing} lies in the affine span of {eta}")
    return v / norm


def search_direction(ns: NodeSet, sigma, eta):
    """Outward direction of edge ``eta`` of vertex ``sigma`` (raycast.py:320-342)."""
    extra = set(sigma) - set(eta)
    if len(extra) != 1 or not set(eta) <= set(sigma):
        raise ValueError("eta must be sigma minus exactly one generator")
    return _search_direction(ns.points, tuple(eta), extra.pop())


def vertex_directions_batch(ns: NodeSet, sigma):
    """All d+1 edge directions of many vertices on the GPU (vr_vertex_directions).

    Returns (u (V, d+1, d) device tensor, ok (V, d+1) uint8 device tensor)."""
    rec, _ = ns.device_records()
    dev = rec.device
    L = _lib.lib()
    sd = _as_dev(sigma if isinstance(sigma, torch.Tensor) else np.asarray(sigma), dev,
                 torch.int32).view(-1, ns.dim + 1)
    nv = sd.shape[0]
    u = torch.empty((nv, ns.dim + 1, ns.dim), dtype=torch.float64, device=dev)
    ok = torch.empty((nv, ns.dim + 1), dtype=torch.uint8, device=dev)
    _lib.check(L.vr_vertex_directions(_lib.ptr(rec), ns.dim, _lib.ptr(sd), nv, _lib.ptr(u),
                                      _lib.ptr(ok), _lib.stream_handle()), "vr_vertex_directions")
    return u, ok


def _vertex_directions(pts, sigma, positions):
    """Outward directions for several edges of one vertex (raycast.py:345-378).

    Host fp64 inverse with the reference's column convention; the traversal
    itself uses the batched device kernel (vr_vertex_directions)."""
    sub = pts[list(sigma)]
    diffs = sub[1:] - sub[0]
    try:
        inv = np.linalg.inv(diffs)
    except np.linalg.LinAlgError:
        raise DegenerateConfiguration(f"generators of {sigma} are affinely dependent") from None
    out = {}
    for k in positions:
        v = inv.sum(axis=1) if k == 0 else -inv[:, k - 1]
        norm = math.sqrt(float(v @ v))
        if not norm > 0.0 or not math.isfinite(norm):
            raise DegenerateConfiguration(f"generators of {sigma} are affinely dependent")
        out[k] = v / norm
    return out


class HostRaycaster:
    """Batched RayCast on host (pinned) arrays.  Chunks cycle through `nbuf`
    device buffers; H2D copies, D2H copies and kernels run on separate
    streams (several compute streams, so one chunk's kernel tail overlaps the
    next chunk's kernel) -- the copy engines and the SMs work concurrently.
    Each chunk's device work replays a captured CUDA graph.  The end-to-end
    public entry point for callers whose rays live in host memory.  Defaults
    (chunks growing 32k -> 256k rays and a 32k last chunk, 8 buffers, 4
    compute streams) were picked with tools/e2e_timeline.py on the config-2
    rays: chunks are sorted independently, and a chunk's rays are sparser
    than the whole batch's (less warp coherence), so the chunked pipeline
    trades some kernel efficiency for overlapping the copies."""

    def __init__(self, ns: NodeSet, n_max: int, eta_len: int, chunk: int = 1 << 18,
                 min_chunk: int = 1 << 15, graphs: bool = True, nbuf: int = 8,
                 compute_streams: int = 4):
        rec, _ = ns.device_records()
        self.ns, self.dev, self.k = ns, rec.device, int(eta_len)
        self.chunk = max(1, min(int(chunk), int(n_max)))  # device buffers hold one chunk
        self.min_chunk = max(1, min(int(min_chunk), self.chunk))
        d = ns.dim
        c = self.chunk
        self.h2d_stream = torch.cuda.Stream(self.dev)
        self.NBUF = max(int(nbuf), int(compute_streams))
        self.comp_streams = [torch.cuda.Stream(self.dev) for _ in range(int(compute_streams))]
        self.d2h_stream = torch.cuda.Stream(self.dev)
        self.buf = [dict(x=torch.empty((c, d), dtype=torch.float64, device=self.dev),
                         u=torch.empty((c, d), dtype=torch.float64, device=self.dev),
                         eta=torch.empty((c, self.k), dtype=torch.int32, device=self.dev),
                         idx=torch.empty(c, dtype=torch.int32, device=self.dev),
                         t=torch.empty(c, dtype=torch.float64, device=self.dev),
                         rp=torch.empty((c, d), dtype=torch.float64, device=self.dev),
                         flag=torch.empty(c, dtype=torch.uint8, device=self.dev),
                         h2d=torch.cuda.Event(), done=torch.cuda.Event(), d2h=torch.cuda.Event())
                    for _ in range(self.NBUF)]
        # Each buffer's workspace is sized for a full chunk here, so a later
        # (larger) chunk never reallocates a buffer an earlier captured graph
        # still points at.
        self.ws = [Workspace() for _ in range(self.NBUF)]
        nbytes = ctypes.c_int64(0)
        L = _lib.lib()
        if ns.fast_paths:
            _lib.check(L.vr_ray_order(None, None, d, 1, None, c, d, ns.n, None, None,
                                      ctypes.byref(nbytes), None), "vr_ray_order (size)")
        for w in self.ws:
            w.get("recheck_list", (c,), torch.int32, self.dev)
            w.get("recheck_count", (1,), torch.int32, self.dev)
            w.get("order", (c,), torch.int32, self.dev)
            w.get("order_tmp", (max(1, nbytes.value),), torch.uint8, self.dev)
        # One CUDA graph per (buffer, chunk size, mode, screen): the per-chunk
        # work (ray order, pruned RayCast, exact re-check) replays without the
        # ~0.5 ms of host-side launch overhead, so small chunks (short
        # pipeline fill and drain) become affordable.
        self.use_graphs = bool(graphs)
        self._graphs = {}

    def _compute(self, bi, m, cs, stats, mode, screen):
        b = self.buf[bi]
        args = (self.ns, b["x"][:m], b["u"][:m], b["eta"][:m])
        kw = dict(out=dict(idx=b["idx"][:m], t=b["t"][:m], rp=b["rp"][:m], flag=b["flag"][:m]),
                  workspace=self.ws[bi], stream=cs, mode=mode, screen=screen)
        key = (bi, m, mode, screen)
        g = self._graphs.get(key) if self.use_graphs else None
        if g is not None:
            g.replay()
            if stats is not None:
                stats.add(m)
            return
        raycast_batch(*args, stats=stats, **kw)  # eager (also the capture warm-up)
        if self.use_graphs:
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, stream=cs):
                    raycast_batch(*args, **kw)
            except RuntimeError:  # capture unsupported here: stay eager (same kernels)
                self.use_graphs = False
                return
            self._graphs[key] = g

    def schedule(self, n):
        """Chunk bounds: sizes grow geometrically from min_chunk to chunk and
        the last chunk is small again, so the first kernel starts after a
        short H2D copy and the final D2H copy is short (pipeline fill and
        drain), while the middle chunks keep the SMs full."""
        out, lo, size = [], 0, self.min_chunk
        while lo < n:
            rest = n - lo
            if rest <= size + self.min_chunk:
                # tail: split the remainder so the last piece is ~min_chunk
                tail = self.min_chunk if rest > 2 * self.min_chunk else \
                    (rest // 2 if rest > self.chunk else 0)
                if tail:
                    out.append((lo, n - tail))
                    lo = n - tail
                out.append((lo, n))
                break
            out.append((lo, lo + size))
            lo += size
            size = min(2 * size, self.chunk)
        return out

    @staticmethod
    def pinned(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True)

    def run(self, hx, hu, heta, hidx, ht, hrp, hflag, stats=None, mode="auto", screen="fp32",
            sync=True, trace=None):
        """hx, hu (n, d) f64, heta (n, k) i32 pinned inputs; outputs pinned
        hidx (n,) i32, ht (n,) f64, hrp (n, d) f64, hflag (n,) u8.  Returns
        after the last D2H copy has completed.  `trace` (a list) receives
        (chunk size, h2d-done, compute-done, d2h-done) CUDA events per chunk
        after a start event (tools/e2e_probe.py timelines)."""
        n = hx.shape[0]
        if trace is not None:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(self.h2d_stream)
            trace.append(ev0)

        def mark(stream):
            if trace is None:
                return None
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e
        if self.ns.n >= PRUNE_MIN_GENERATORS and mode != "exhaustive" and self.ns.fast_paths:
            self.ns.prune_index(self.dev)
        if screen == "fp32":
            self.ns.screen32(self.dev)
        for ci, (lo, hi) in enumerate(self.schedule(n)):
            b = self.buf[ci % self.NBUF]
            cs = self.comp_streams[ci % len(self.comp_streams)]
            m = hi - lo
            with torch.cuda.stream(self.h2d_stream):
                if ci >= self.NBUF:
                    self.h2d_stream.wait_event(b["d2h"])  # buffer drained
                b["x"][:m].copy_(hx[lo:hi], non_blocking=True)
                b["u"][:m].copy_(hu[lo:hi], non_blocking=True)
                b["eta"][:m].copy_(heta[lo:hi], non_blocking=True)
                b["h2d"].record(self.h2d_stream)
                e1 = mark(self.h2d_stream)
            with torch.cuda.stream(cs):
                cs.wait_event(b["h2d"])
                self._compute(ci % self.NBUF, m, cs, stats, mode, screen)
                b["done"].record(cs)
                e2 = mark(cs)
            with torch.cuda.stream(self.d2h_stream):
                self.d2h_stream.wait_event(b["done"])
                hidx[lo:hi].copy_(b["idx"][:m], non_blocking=True)
                ht[lo:hi].copy_(b["t"][:m], non_blocking=True)
                hrp[lo:hi].copy_(b["rp"][:m], non_blocking=True)
                hflag[lo:hi].copy_(b["flag"][:m], non_blocking=True)
                b["d2h"].record(self.d2h_stream)
                if trace is not None:
                    trace.append((m, e1, e2, mark(self.d2h_stream)))
        if sync:
            self.d2h_stream.synchronize()
