"""Monte-Carlo cell volumes and interface areas on the B200.

Drop-in for pkg/src/voronray/integrate_mc.py.  Every ray is the RayCast from
the cell generator with eta = (i,) (integrate_mc.py:60-67); the per-cell sums
of l^d and l^(d-1)/cos(n_ij, y) (integrate_mc.py:147-160) are formed on the
device in ray order by vr_mc_reduce.

Two direction sources:

* ``mc_areas_only(ns, i, n, rng)`` -- the reference signature: directions are
  drawn from the caller's ``rng`` on the host in the reference order
  (``rng.standard_normal((n, d))`` == n draws of ``(d,)``), so results agree
  with the reference to floating-point roundoff;
* ``mc_cells(ns, cells, n, seed)`` -- the throughput path: Philox4x32-10
  directions generated inside the kernel, keyed by (seed, cell, ray), so the
  result does not depend on launch shape or GPU count.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import _lib
from .core import NodeSet
from .errors import DegenerateConfiguration, UnboundedRay
from .raycast import (RaycastStats, Workspace, _screen, _use_pruned, candidate_records,
                      ray_order)

Integrand = Callable[[np.ndarray], float]

CELL_OK, CELL_UNBOUNDED, CELL_DEGENERATE, CELL_OVERFLOW = 0, 1, 2, 3


@dataclass
class CellIntegrals:
    """Per-cell results (integrate_mc.py:27-41)."""

    volume: float = 0.0
    area: dict = field(default_factory=dict)
    surface_integral: dict = field(default_factory=dict)
    volume_integral: float = 0.0
    n_rays: int = 0
    m_subsamples: int = 0


def sphere_surface_area(d: int) -> float:
    """2 pi^(d/2) / Gamma(d/2) (integrate_mc.py:44-48)."""
    if d < 1:
        raise ValueError("dimension must be positive")
    return 2.0 * math.pi ** (d / 2.0) / math.gamma(d / 2.0)


def sample_unit_sphere(d: int, rng) -> np.ndarray:
    """Uniform direction by normalising a Gaussian draw (integrate_mc.py:51-56)."""
    while True:
        y = rng.standard_normal(d)
        norm = math.sqrt(float(y @ y))
        if norm > 0.0:
            return y / norm


@dataclass
class MCResult:
    """Batched MC output for cells[c]: volume, faces sorted by neighbour."""

    cells: np.ndarray
    volume: np.ndarray
    face_offsets: np.ndarray
    face_j: np.ndarray
    face_area: np.ndarray
    status: np.ndarray
    first_bad: np.ndarray
    samples: np.ndarray = None

    def areas(self, c):
        lo, hi = self.face_offsets[c], self.face_offsets[c + 1]
        return {int(j): float(a) for j, a in zip(self.face_j[lo:hi], self.face_area[lo:hi])}


MC_ORDER_RAYS = True  # direction-sorted processing order in the pruned MC path


def _mc_device(ns: NodeSet, cells, n, dirs=None, seed=0, candidates=None, max_faces=256,
               degenerate_is_error=True, want_samples=False, workspace=None, stats=None,
               mode="auto", screen="fp32", work=None):
    """Run rays + recheck + reduce for len(cells) cells x n rays; device tensors out."""
    rec, sqmax = ns.device_records()
    dev = rec.device
    L = _lib.lib()
    d = ns.dim
    cells_d = torch.as_tensor(np.ascontiguousarray(cells, dtype=np.int32), device=dev) \
        if not isinstance(cells, torch.Tensor) else cells.to(device=dev, dtype=torch.int32).contiguous()
    nc = cells_d.shape[0]
    total = nc * n
    ws = workspace or Workspace()
    dd = None
    if dirs is not None:
        dd = dirs if isinstance(dirs, torch.Tensor) else torch.as_tensor(
            np.ascontiguousarray(dirs, dtype=np.float64))
        dd = dd.to(device=dev, dtype=torch.float64).contiguous().view(total, d)
    cand = crec = None
    n_cand = 0
    s32 = _screen(ns, dev, screen)
    if candidates is not None:
        cand, crec, s32 = candidate_records(ns, candidates, dev, screen)
        n_cand = cand.shape[0]
    s32p = ctypes.byref(s32.struct) if s32 is not None else None
    idx = ws.get("mc_idx", (total,), torch.int32, dev)
    t = ws.get("mc_t", (total,), torch.float64, dev)
    flag = ws.get("mc_flag", (total,), torch.uint8, dev)
    rl = ws.get("mc_rl", (total,), torch.int32, dev)
    rc = ws.get("mc_rc", (1,), torch.int32, dev)
    sh = _lib.stream_handle()
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    if _use_pruned(ns, candidates, mode):
        ix = ns.prune_index(dev)
        order = None
        if MC_ORDER_RAYS and n >= 32:
            # Rays of one cell share their origin; sorting them by direction
            # class makes the 32 rays of a warp coherent (smaller union of
            # spheres, fewer tree nodes).  The Philox directions are
            # materialised once so the order can be computed; results are
            # independent of the order.
            if dd is None:
                dd = ws.get("mc_dirs", (total, d), torch.float64, dev)
                _lib.check(L.vr_mc_directions(d, nc, _lib.ptr(cells_d), n, seed, _lib.ptr(dd), sh),
                           "vr_mc_directions")
            order = ray_order(dd.view(total, d), rays_per_cell=n, n_base=nc, workspace=ws)
        _lib.check(L.vr_mc_rays_pruned(_lib.ptr(rec), ns.n, d, sqmax, s32p, ctypes.byref(ix.struct),
                                       _lib.ptr(cells_d), nc, n, _lib.ptr(dd), seed, _lib.ptr(order),
                                       _lib.ptr(idx), _lib.ptr(t), _lib.ptr(flag), _lib.ptr(rl),
                                       _lib.ptr(rc), _lib.ptr(work), sh), "vr_mc_rays_pruned")
    else:
        _lib.check(L.vr_mc_rays(_lib.ptr(rec), ns.n, d, sqmax, s32p, _lib.ptr(crec), _lib.ptr(cand),
                                n_cand, _lib.ptr(cells_d), nc, n, _lib.ptr(dd), seed,
                                _lib.ptr(idx), _lib.ptr(t), _lib.ptr(flag), _lib.ptr(rl),
                                _lib.ptr(rc), sh), "vr_mc_rays")
    _lib.check(L.vr_mc_recheck(_lib.ptr(rec), ns.n, d, _lib.ptr(crec), _lib.ptr(cand), n_cand,
                               _lib.ptr(cells_d), n, _lib.ptr(dd), seed, _lib.ptr(rl),
                               _lib.ptr(rc), total, _lib.ptr(idx), _lib.ptr(t), _lib.ptr(flag),
                               sh), "vr_mc_recheck")
    vol = torch.empty(nc, dtype=torch.float64, device=dev)
    fj = torch.empty((nc, max_faces), dtype=torch.int32, device=dev)
    fa = torch.empty((nc, max_faces), dtype=torch.float64, device=dev)
    nf = torch.empty(nc, dtype=torch.int32, device=dev)
    st = torch.empty(nc, dtype=torch.int32, device=dev)
    fb = torch.empty(nc, dtype=torch.int64, device=dev)
    smp = torch.empty(total, dtype=torch.float64, device=dev) if want_samples else None
    mb = int(L.vr_mc_map_bytes(nc, max_faces, 0))  # > 0 only past the shared-memory face map
    mws = ws.get("mc_map", (mb,), torch.uint8, dev) if mb else None
    _lib.check(L.vr_mc_reduce(_lib.ptr(rec), d, _lib.ptr(cells_d), nc, n, _lib.ptr(dd), seed,
                              _lib.ptr(idx), _lib.ptr(t), _lib.ptr(flag), max_faces,
                              1 if degenerate_is_error else 0, sphere_surface_area(d),
                              None, 0, _lib.ptr(mws), mb,
                              _lib.ptr(vol), _lib.ptr(fj), _lib.ptr(fa), _lib.ptr(nf),
                              _lib.ptr(st), _lib.ptr(fb), _lib.ptr(smp), sh), "vr_mc_reduce")
    if stats is not None:
        stats.add(total)
    # faces of a cell are bounded by its rays and by its possible neighbours
    bound = max(1, min(n, n_cand if candidates is not None else ns.n - 1))

    def rereduce(rows):
        """Reduce the cell rows `rows` again with a face table large enough
        for any cell (the reference's face dict is unbounded,
        integrate_mc.py:147-160); the ray results are reused."""
        m = len(rows)
        sel = torch.as_tensor(np.ascontiguousarray(rows, dtype=np.int32), device=dev)
        mb = int(L.vr_mc_map_bytes(m, bound, 0))
        mws = torch.empty(mb, dtype=torch.uint8, device=dev) if mb else None
        o = dict(volume=torch.empty(m, dtype=torch.float64, device=dev),
                 face_j=torch.empty((m, bound), dtype=torch.int32, device=dev),
                 face_area=torch.empty((m, bound), dtype=torch.float64, device=dev),
                 nfaces=torch.empty(m, dtype=torch.int32, device=dev),
                 status=torch.empty(m, dtype=torch.int32, device=dev),
                 first_bad=torch.empty(m, dtype=torch.int64, device=dev))
        _lib.check(L.vr_mc_reduce(_lib.ptr(rec), d, _lib.ptr(cells_d), nc, n, _lib.ptr(dd), seed,
                                  _lib.ptr(idx), _lib.ptr(t), _lib.ptr(flag), bound,
                                  1 if degenerate_is_error else 0, sphere_surface_area(d),
                                  _lib.ptr(sel), m, _lib.ptr(mws), mb,
                                  _lib.ptr(o["volume"]), _lib.ptr(o["face_j"]),
                                  _lib.ptr(o["face_area"]), _lib.ptr(o["nfaces"]),
                                  _lib.ptr(o["status"]), _lib.ptr(o["first_bad"]), None,
                                  _lib.stream_handle()), "vr_mc_reduce (large faces)")
        return o

    return dict(volume=vol, face_j=fj, face_area=fa, nfaces=nf, status=st, first_bad=fb,
                samples=smp, ray_idx=idx, ray_t=t, ray_flag=flag, rereduce=rereduce,
                max_faces=max_faces, face_bound=bound)


def _collect(cells, out, want_samples):
    """Compact the per-cell face tables on the device (cells x max_faces ->
    the faces actually hit, CSR order) before the host copy.  Cells whose
    faces overflowed the table are reduced again with a table large enough
    for any cell (out["rereduce"]) and spliced in, so no cell is lost."""
    nf_d = out["nfaces"]
    fj_d, fa_d = out["face_j"], out["face_area"]
    status = _lib.to_host(out["status"]).copy()
    ovf = np.nonzero(status == CELL_OVERFLOW)[0]
    if ovf.size and out.get("rereduce") is not None and out["face_bound"] > out["max_faces"]:
        nf_d = nf_d.clone()
        nf_d[torch.as_tensor(ovf, device=nf_d.device)] = 0
    mask = torch.arange(fj_d.shape[1], device=fj_d.device)[None, :] < nf_d[:, None]
    nf = _lib.to_host(nf_d).astype(np.int64)
    face_j = _lib.to_host(fj_d[mask])
    face_area = _lib.to_host(fa_d[mask])
    volume = _lib.to_host(out["volume"]).copy()
    first_bad = _lib.to_host(out["first_bad"]).copy()
    if ovf.size and out.get("rereduce") is not None and out["face_bound"] > out["max_faces"]:
        r = out["rereduce"](ovf)
        rn = _lib.to_host(r["nfaces"]).astype(np.int64)
        rmask = torch.arange(r["face_j"].shape[1], device=fj_d.device)[None, :] < r["nfaces"][:, None]
        rj, ra = _lib.to_host(r["face_j"][rmask]), _lib.to_host(r["face_area"][rmask])
        nf[ovf] = rn
        status[ovf] = _lib.to_host(r["status"])
        first_bad[ovf] = _lib.to_host(r["first_bad"])
        volume[ovf] = _lib.to_host(r["volume"])
        owner = np.repeat(np.arange(len(nf)), nf)
        big = np.zeros(len(nf), dtype=bool)
        big[ovf] = True
        sel = big[owner]
        fj_all = np.empty(owner.size, dtype=np.int32)
        fa_all = np.empty(owner.size, dtype=np.float64)
        fj_all[~sel], fa_all[~sel] = face_j, face_area
        fj_all[sel], fa_all[sel] = rj, ra
        face_j, face_area = fj_all, fa_all
    off = np.zeros(len(nf) + 1, dtype=np.int64)
    np.cumsum(nf, out=off[1:])
    return MCResult(cells=np.asarray(cells), volume=volume, face_offsets=off,
                    face_j=face_j, face_area=face_area, status=status.astype(np.int32),
                    first_bad=first_bad,
                    samples=_lib.to_host(out["samples"]) if want_samples else None)


def mc_cells(ns: NodeSet, cells, n: int, seed: int = 0, max_faces: int = 256,
             want_samples=False, stats: RaycastStats = None, chunk_rays: int = 1 << 26,
             mode="auto", screen="fp32", work=None):
    """Batched device MC (Philox directions) over many cells.

    Returns an :class:`MCResult`; cells whose status is not CELL_OK are the
    ones the reference would reject (UnboundedRay / DegenerateConfiguration).
    Work is split into chunks of at most ``chunk_rays`` rays.
    """
    if n < 1:
        raise ValueError("need n >= 1 rays")
    if max_faces < 1:
        raise ValueError("max_faces must be positive")
    cells = np.ascontiguousarray(cells, dtype=np.int32)
    per_chunk = max(1, chunk_rays // n)
    parts = []
    ws = Workspace()
    for lo in range(0, len(cells), per_chunk):
        sub = cells[lo:lo + per_chunk]
        out = _mc_device(ns, sub, n, seed=seed, max_faces=max_faces, want_samples=want_samples,
                         workspace=ws, stats=stats, mode=mode, screen=screen, work=work)
        parts.append(_collect(sub, out, want_samples))
    if len(parts) == 1:
        return parts[0]
    off = [np.zeros(1, dtype=np.int64)]
    base = 0
    for p in parts:
        off.append(p.face_offsets[1:] + base)
        base += p.face_offsets[-1]
    return MCResult(cells=cells, volume=np.concatenate([p.volume for p in parts]),
                    face_offsets=np.concatenate(off),
                    face_j=np.concatenate([p.face_j for p in parts]),
                    face_area=np.concatenate([p.face_area for p in parts]),
                    status=np.concatenate([p.status for p in parts]),
                    first_bad=np.concatenate([p.first_bad for p in parts]),
                    samples=np.concatenate([p.samples for p in parts]) if want_samples else None)


def mc_directions(ns_dim: int, cells, n: int, seed: int = 0, device=None):
    """The raw Gaussian draws the Philox path uses for (cells x n) rays,
    shape (len(cells) * n, d) -- for replay into a host consumer."""
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    cd = torch.as_tensor(np.ascontiguousarray(cells, dtype=np.int32), device=dev)
    out = torch.empty((len(cells) * n, ns_dim), dtype=torch.float64, device=dev)
    _lib.check(L.vr_mc_directions(ns_dim, len(cells), _lib.ptr(cd), n,
                                  int(seed) & 0xFFFFFFFFFFFFFFFF, _lib.ptr(out),
                                  _lib.stream_handle()), "vr_mc_directions")
    return out.cpu().numpy()


def _max_faces_for(ns, n, neighbors):
    """Face-table width that no cell can overflow: distinct faces are
    bounded by the rays and by the possible neighbours."""
    if neighbors is not None:
        return max(1, min(len(neighbors), n))
    return max(1, min(n, ns.n - 1))


def mc_areas_only(ns: NodeSet, i: int, n: int, rng, neighbors=None,
                  stats: RaycastStats = None, return_samples: bool = False):
    """Face areas and volume of cell i (integrate_mc.py:124-161).

    Returns ``(areas, volume)`` or ``(areas, volume, samples)``.  Raises
    :class:`UnboundedRay` (with the unit direction of the first escaping ray)
    or :class:`DegenerateConfiguration` like the reference per-ray path; with
    ``neighbors`` the degeneracy band is not checked, like _mc_areas_batch.
    """
    if n < 1:
        raise ValueError("need n >= 1 rays")
    d = ns.dim
    if neighbors is not None and len(neighbors) == 0:
        # reference: an empty candidate list makes every probe all-invalid, so
        # the first ray escapes (integrate_mc.py:143-146 -> _cast, raycast.py:100-117)
        raise UnboundedRay(i, sample_unit_sphere(d, rng))
    z = np.asarray(rng.standard_normal((n, d)), dtype=np.float64).reshape(n, d)
    use_nb = neighbors is not None and len(neighbors) > 0
    max_faces = _max_faces_for(ns, n, neighbors if use_nb else None)
    out = _mc_device(ns, [int(i)], n, dirs=z, candidates=neighbors if use_nb else None,
                     max_faces=max_faces, degenerate_is_error=not use_nb,
                     want_samples=True, stats=stats)
    res = _collect([i], out, True)
    st = int(res.status[0])
    if st == CELL_UNBOUNDED:
        y = z[int(res.first_bad[0])]
        raise UnboundedRay(i, y / math.sqrt(float(y @ y)))
    if st == CELL_DEGENERATE:
        raise DegenerateConfiguration(f"a foreign generator lies on a circumsphere of cell {i}")
    areas = res.areas(0)
    volume = float(res.volume[0])
    return (areas, volume, res.samples) if return_samples else (areas, volume)


def _draw_integrate_stream(rng, n, m, d):
    """Directions and subsample positions in the reference's RNG order
    (integrate_mc.py:341-355): per ray one sample_unit_sphere draw (raw
    normals, redrawn while the norm is 0), then m uniforms."""
    z = np.empty((n, d))
    u = np.empty((n, m))
    for k in range(n):
        while True:
            y = np.asarray(rng.standard_normal(d), dtype=float)
            if math.sqrt(float(y @ y)) > 0.0:
                break
        z[k] = y
        for s in range(m):
            u[k, s] = rng.random()
    return z, u


def _integrate_device(ns, cells, n, m, kind, coef, dirs=None, unif=None, seed=0,
                      candidates=None, max_faces=256, stats=None, workspace=None):
    L = _lib.lib()
    out = _mc_device(ns, cells, n, dirs=dirs, seed=seed, candidates=candidates,
                     max_faces=max_faces, degenerate_is_error=True, stats=stats,
                     workspace=workspace)
    rec, _ = ns.device_records()
    dev = rec.device
    d = ns.dim
    cells_d = torch.as_tensor(np.ascontiguousarray(cells, dtype=np.int32), device=dev)
    nc = cells_d.shape[0]
    dd = None if dirs is None else torch.as_tensor(
        np.ascontiguousarray(dirs, dtype=np.float64), device=dev)
    ud = None if unif is None else torch.as_tensor(
        np.ascontiguousarray(unif, dtype=np.float64), device=dev)
    cf = (ctypes.c_double * 9)(*(list(coef) + [0.0] * (9 - len(coef))))  # host array
    vol = torch.empty(nc, dtype=torch.float64, device=dev)
    fj = torch.empty((nc, max_faces), dtype=torch.int32, device=dev)
    fa = torch.empty((nc, max_faces), dtype=torch.float64, device=dev)
    fs = torch.empty((nc, max_faces), dtype=torch.float64, device=dev)
    vi = torch.empty(nc, dtype=torch.float64, device=dev)
    nf = torch.empty(nc, dtype=torch.int32, device=dev)
    st = torch.empty(nc, dtype=torch.int32, device=dev)
    fb = torch.empty(nc, dtype=torch.int64, device=dev)
    mb = int(L.vr_mc_map_bytes(nc, max_faces, 1))
    mws = torch.empty(mb, dtype=torch.uint8, device=dev) if mb else None
    _lib.check(L.vr_mc_integrate(_lib.ptr(rec), d, _lib.ptr(cells_d), nc, n, _lib.ptr(dd),
                                 int(seed) & 0xFFFFFFFFFFFFFFFF, _lib.ptr(out["ray_idx"]),
                                 _lib.ptr(out["ray_t"]), _lib.ptr(out["ray_flag"]), max_faces,
                                 sphere_surface_area(d), int(kind), cf, int(m),
                                 _lib.ptr(ud), None, 0, _lib.ptr(mws), mb,
                                 _lib.ptr(vol), _lib.ptr(fj), _lib.ptr(fa),
                                 _lib.ptr(fs), _lib.ptr(vi), _lib.ptr(nf), _lib.ptr(st),
                                 _lib.ptr(fb), _lib.stream_handle()), "vr_mc_integrate")
    if max_faces < out["face_bound"] and bool((st == CELL_OVERFLOW).any()):
        # a cell hit more faces than the table holds: redo the reduction with
        # a table no cell can overflow (the reference's face dict is unbounded)
        return _integrate_device(ns, cells, n, m, kind, coef, dirs=dirs, unif=unif, seed=seed,
                                 candidates=candidates, max_faces=out["face_bound"],
                                 stats=None, workspace=workspace)
    return dict(volume=vol.cpu().numpy(), face_j=fj.cpu().numpy(), face_area=fa.cpu().numpy(),
                face_surf=fs.cpu().numpy(), vol_integral=vi.cpu().numpy(),
                nfaces=nf.cpu().numpy(), status=st.cpu().numpy(), first_bad=fb.cpu().numpy(),
                ray_idx=out["ray_idx"], ray_t=out["ray_t"], ray_flag=out["ray_flag"])


def mc_integrate_cell(ns: NodeSet, i: int, f: Integrand, n: int, m: int, rng,
                      neighbors=None, stats: RaycastStats = None) -> CellIntegrals:
    """Volume, face areas, and surface / volume integrals of cell i
    (integrate_mc.py:70-121), same RNG consumption order as the reference.

    Every ray is cast on the GPU.  Built-in integrands
    (:mod:`paper_2405_10050_b200.integrands`) are evaluated in the reduction
    kernel; any other Python callable is evaluated on the host in the
    reference's order (it is user code).

    Raises:
        UnboundedRay: a ray escaped (first escaping direction attached).
    """
    if n < 1 or m < 1:
        raise ValueError("need n >= 1 rays and m >= 1 subsamples")
    d = ns.dim
    if neighbors is not None and len(neighbors) == 0:
        raise UnboundedRay(i, sample_unit_sphere(d, rng))  # as mc_areas_only
    z, unif = _draw_integrate_stream(rng, n, m, d)
    cand = neighbors if neighbors is not None and len(neighbors) > 0 else None
    max_faces = _max_faces_for(ns, n, cand)
    spec = getattr(f, "device_spec", None)
    if spec is not None:
        res = _integrate_device(ns, [int(i)], n, m, spec[0], spec[1], dirs=z, unif=unif,
                                candidates=cand, max_faces=max_faces, stats=stats)
        st = int(res["status"][0])
        if st == CELL_UNBOUNDED:
            y = z[int(res["first_bad"][0])]
            raise UnboundedRay(i, y / math.sqrt(float(y @ y)))
        if st == CELL_DEGENERATE:
            raise DegenerateConfiguration(f"a foreign generator lies on a circumsphere of cell {i}")
        k = int(res["nfaces"][0])
        js = [int(j) for j in res["face_j"][0, :k]]
        return CellIntegrals(volume=float(res["volume"][0]),
                             area={j: float(a) for j, a in zip(js, res["face_area"][0, :k])},
                             surface_integral={j: float(s) for j, s in
                                               zip(js, res["face_surf"][0, :k])},
                             volume_integral=float(res["vol_integral"][0]), n_rays=n,
                             m_subsamples=m)
    # generic callable: hits from the GPU, integrand sums on the host in ray order
    out = _mc_device(ns, [int(i)], n, dirs=z, candidates=cand, max_faces=max_faces,
                     degenerate_is_error=True, stats=stats)
    idx = out["ray_idx"].cpu().numpy()
    t = out["ray_t"].cpu().numpy()
    flag = out["ray_flag"].cpu().numpy()
    pts = ns.points
    xi = pts[i]
    area, fsurf = {}, {}
    vol = fvol = 0.0
    for k in range(n):
        y = z[k] / math.sqrt(float(z[k] @ z[k]))
        if flag[k] == 1:
            raise UnboundedRay(i, y)
        if flag[k] == 3:
            raise DegenerateConfiguration(f"a foreign generator lies on a circumsphere of cell {i}")
        j = int(idx[k])
        rp = xi + t[k] * y
        seg = rp - xi
        length = math.sqrt(float(seg @ seg))
        nij = pts[j] - xi
        cosang = float(nij @ y) / math.sqrt(float(nij @ nij))
        w = length ** (d - 1) / cosang
        area[j] = area.get(j, 0.0) + w
        fsurf[j] = fsurf.get(j, 0.0) + f(rp) * w
        vol += length ** d
        acc = 0.0
        for s in range(m):
            ts = unif[k, s]
            acc += f(xi + ts * seg) * ts ** (d - 1)
        fvol += acc * length ** d
    surf = sphere_surface_area(d)
    scale = surf / n
    return CellIntegrals(volume=vol * surf / (d * n), area={j: a * scale for j, a in area.items()},
                         surface_integral={j: s * scale for j, s in fsurf.items()},
                         volume_integral=fvol * surf / (n * m), n_rays=n, m_subsamples=m)


def mc_integrals_cells(ns: NodeSet, cells, n: int, m: int, f, seed: int = 0,
                       max_faces: int = 256):
    """Batched device MC integrals for a built-in integrand: Philox
    directions and subsample positions, everything on the GPU.  Returns a
    dict of per-cell arrays (volume, vol_integral, status, faces...)."""
    spec = getattr(f, "device_spec", None)
    if spec is None:
        raise ValueError("mc_integrals_cells needs a built-in integrand (integrands.py)")
    return _integrate_device(ns, np.asarray(cells, dtype=np.int32), n, m, spec[0], spec[1],
                             seed=seed, max_faces=max_faces)


def mc_uniforms(cells, n: int, m: int, seed: int = 0, device=None):
    """The Philox subsample uniforms of mc_integrals_cells, (len(cells)*n, m)."""
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    cd = torch.as_tensor(np.ascontiguousarray(cells, dtype=np.int32), device=dev)
    out = torch.empty((len(cells) * n, m), dtype=torch.float64, device=dev)
    _lib.check(L.vr_mc_uniforms(len(cells), _lib.ptr(cd), n, m, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                _lib.ptr(out), _lib.stream_handle()), "vr_mc_uniforms")
    return out.cpu().numpy()
