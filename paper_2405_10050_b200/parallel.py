"""Multi-GPU sharding: one process per GPU, torch.distributed
(NCCL over NVLink on B200 boxes, gloo for CPU tests) for the plumbing.

* Batched RayCast / MC: rays and cells are independent units.  Each rank
  takes a contiguous shard, generators are replicated, nothing crosses the
  link on the data path; results are gathered once at the end.  MC
  directions are keyed by (seed, cell, ray), so the answer does not depend on
  the number of ranks.
* Traversal (``ShardedTraversal``): owner-sharded tables.  Vertex sigma lives
  on rank owner(sigma), edge eta on owner(eta) (a hash of the sorted tuple);
  per level every rank raycasts the open edges of its OWN frontier, sends
  each hit sigma' to its owner (one all-to-all), the owners dedupe and store
  the new vertices, and the new vertices' d+1 edge keys go to the edge
  owners (a second all-to-all), which bump them and answer with the counts
  (the reply), which are the next level's open test (graph.py:115-135).
  Tables, vertex arrays and raycasts all scale with the rank count; the
  result is the single-GPU level-synchronous traversal's for any rank count.
  ``ShardedRaycast`` (replicated tables, ray-sharded levels, one all-gather
  of the hits) is kept for reference.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world():
    """(world_size, rank) of the default group, (1, 0) when not initialised."""
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def shard_bounds(n, size, rank):
    """Contiguous [lo, hi) shard of n units for `rank` of `size` (balanced)."""
    base, extra = divmod(int(n), int(size))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allgather_rows(t, group=None):
    """All-gather row blocks of different lengths (concatenated in rank
    order).  Works for NCCL (cuda tensors) and gloo (cpu tensors)."""
    size = dist.get_world_size(group)
    if size == 1:
        return t
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(size)]
    dist.all_gather(ns, n, group=group)
    counts = [int(v.item()) for v in ns]
    m = max(counts)
    pad = torch.zeros((m - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    tp = torch.cat([t, pad]) if m > t.shape[0] else t.contiguous()
    outs = [torch.empty_like(tp) for _ in range(size)]
    dist.all_gather(outs, tp, group=group)
    return torch.cat([o[:c] for o, c in zip(outs, counts)])


class ShardedRaycast:
    """Wrap a per-rank raycast ``fn(x, u, eta) -> (idx int32, flag uint8)``:
    every rank passes the SAME full ray arrays, computes its shard, and gets
    the full result back (one all-gather of 5 bytes per ray)."""

    def __init__(self, fn, group=None):
        self.fn, self.group = fn, group

    def __call__(self, x, u, eta):
        size = dist.get_world_size(self.group) if dist.is_initialized() else 1
        rank = dist.get_rank(self.group) if dist.is_initialized() else 0
        lo, hi = shard_bounds(x.shape[0], size, rank)
        idx, flag = self.fn(x[lo:hi], u[lo:hi], eta[lo:hi])
        if size == 1:
            return idx, flag
        packed = torch.cat([idx.to(torch.int32).view(-1, 1),
                            flag.to(torch.int32).view(-1, 1)], 1)
        full = allgather_rows(packed, self.group)
        return full[:, 0].contiguous(), full[:, 1].to(torch.uint8).contiguous()


def gather_mc(result, group=None, device=None):
    """Gather per-rank MCResult shards (cells in rank order) onto every rank."""
    from .integrate_mc import MCResult
    size = dist.get_world_size(group) if dist.is_initialized() else 1
    if size == 1:
        return result
    dev = device or (torch.device("cuda", torch.cuda.current_device())
                     if torch.cuda.is_available() else torch.device("cpu"))

    def ag(a, dtype):
        return allgather_rows(torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev),
                              group).cpu().numpy()

    nf = np.diff(result.face_offsets)
    cells = ag(result.cells, torch.int64)
    volume = ag(result.volume, torch.float64)
    status = ag(result.status, torch.int64).astype(np.int32)
    first_bad = ag(result.first_bad, torch.int64)
    nf_all = ag(nf, torch.int64)
    face_j = ag(result.face_j, torch.int64).astype(np.int32)
    face_area = ag(result.face_area, torch.float64)
    off = np.zeros(len(nf_all) + 1, dtype=np.int64)
    np.cumsum(nf_all, out=off[1:])
    samples = None
    if result.samples is not None:
        samples = ag(result.samples, torch.float64)
    return MCResult(cells=cells, volume=volume, face_offsets=off, face_j=face_j,
                    face_area=face_area, status=status, first_bad=first_bad, samples=samples)


def mc_cells_sharded(ns, cells, n, seed=0, group=None, **kw):
    """mc_cells over this rank's contiguous shard of `cells`, gathered."""
    from .integrate_mc import mc_cells
    size = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    cells = np.asarray(cells)
    lo, hi = shard_bounds(len(cells), size, rank)
    part = mc_cells(ns, cells[lo:hi], n, seed=seed, **kw)
    return gather_mc(part, group)


def raycast_sharded(ns, x, u, eta, group=None, **kw):
    """raycast_batch on this rank's shard of the rays; full (idx, flag) on
    every rank."""
    from .raycast import raycast_batch

    def fn(xs, us, es):
        r = raycast_batch(ns, xs, us, es, want_rp=False, **kw)
        return r.idx, r.flag

    return ShardedRaycast(fn, group)(x, u, eta)


# ---------------------------------------------------------------------------
# Owner-sharded traversal
# ---------------------------------------------------------------------------

def _exchange(rows, send_counts, group=None):
    """all-to-all of row blocks: rows (n, k) grouped by destination rank with
    send_counts[r] rows for rank r; returns (received rows grouped by source
    rank, recv_counts).  NCCL exchanges device tensors; other backends
    (gloo) stage through host memory."""
    size = dist.get_world_size(group)
    dev = rows.device
    host = dist.get_backend(group) != "nccl"
    cdev = torch.device("cpu") if host else dev
    sc = torch.tensor(list(send_counts), dtype=torch.int64, device=cdev)
    rc = torch.empty(size, dtype=torch.int64, device=cdev)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(v) for v in rc.tolist()]
    k = rows.shape[1]
    src = rows.contiguous().to(cdev)
    out = torch.empty((sum(recv_counts), k), dtype=rows.dtype, device=cdev)
    dist.all_to_all_single(out.view(-1), src.view(-1), [c * k for c in recv_counts],
                           [int(c) * k for c in send_counts], group=group)
    return out.to(dev), recv_counts


def _reply(rows, recv_counts, send_counts, group=None):
    """The reverse exchange: rows (n_recv, k) in the order they were received
    go back to their senders, arriving in each sender's send order."""
    out, _ = _exchange(rows, recv_counts, group)
    return out


class ShardedTraversal:
    """Level-synchronous traversal with owner-sharded vertex / edge tables.

    ``ops`` implements the per-rank table and RayCast operations
    (:class:`DeviceShardOps` on a GPU); the level protocol is here:

    1. rays   -- ops.frontier_rays: open edges of the local frontier (count of
                 the edge < 2, as returned by its owner), their rays, the
                 pruned RayCast (native level driver); escapes are recorded
                 as boundary rays locally;
    2. claim  -- hit sigma' rows -> owner(sigma') (all-to-all); the owner
                 inserts them (smallest received row wins a new key) and
                 stores the new vertices with fresh fp64 circumcentres;
    3. bump   -- the new vertices' d+1 edge keys -> owner(eta) (all-to-all);
                 the owner bumps all keys of the level, then answers each
                 with its count (reverse all-to-all) -> the vertex owner keeps
                 the counts for the next level's open test.
    """

    def __init__(self, ns, ops, group=None):
        self.ns, self.ops, self.group = ns, ops, group
        self.size = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.d = ns.dim
        self.levels = []   # (first local id, end, level)
        self.rays = 0

    def _bucket_exchange(self, rows):
        perm, counts = self.ops.owner_bucket(rows, self.size)
        send = self.ops.gather_rows(rows, perm)
        if self.size == 1:
            return send, perm, counts, counts
        recv, rcounts = _exchange(send, counts, self.group)
        return recv, perm, counts, rcounts

    def _bump(self, first, rows):
        """Edges of the vertices just stored at local ids [first, first + m)."""
        keys = self.ops.vertex_edges(rows)
        recv, perm, counts, rcounts = self._bucket_exchange(keys)
        got = self.ops.bump(recv)                       # (n_recv, 1) counts after all bumps
        back = got if self.size == 1 else _reply(got, rcounts, counts, self.group)
        vals = self.ops.scatter_rows(back, perm, keys.shape[0])
        self.ops.set_counts(first, vals.view(-1, self.d + 1))

    def _global(self, v):
        if self.size == 1:
            return int(v)
        t = torch.tensor([int(v)], dtype=torch.int64,
                         device=self.ops.device if dist.get_backend(self.group) == "nccl"
                         else torch.device("cpu"))
        dist.all_reduce(t, group=self.group)
        return int(t.item())

    def seed(self, sigmas):
        """Distinct seed vertices (the same sorted rows on every rank) at level 0."""
        rows = self.ops.as_rows(sigmas, self.d + 1)
        perm, counts = self.ops.owner_bucket(rows, self.size)
        lo = sum(counts[:self.rank])
        mine = self.ops.gather_rows(rows, perm)[lo:lo + counts[self.rank]]
        first, new = self.ops.add_vertices(mine, None, 0)
        self._bump(first, new)
        self.levels.append((first, first + new.shape[0], 0))
        return self._global(new.shape[0])

    def level(self, lvl, stats=None):
        """One level; returns the number of new vertices over all ranks."""
        f0, f1, _ = self.levels[-1]
        hits = self.ops.frontier_rays(f0, f1, lvl)
        self.rays += hits["n_rays"]
        if stats is not None:
            stats.add(hits["n_rays"])
        cand = hits["sigma"]                              # (n_ok, d + 1) hit sigma'
        recv, _, _, _ = self._bucket_exchange(cand)
        first, new = self.ops.add_vertices(recv, lvl, lvl)
        self._bump(first, new)
        self.levels.append((first, first + new.shape[0], lvl))
        return self._global(new.shape[0])

    def gather(self, with_levels=False):
        """Mesh over the union of the shards (every rank gets all of it)."""
        from .core import Mesh
        a = self.ops.local_arrays()
        lv = torch.zeros(a["sigma"].shape[0], dtype=torch.int32)
        for b, e, level in self.levels:
            lv[b:e] = level
        if self.size > 1:
            host = dist.get_backend(self.group) != "nccl"

            def ag(t):
                src = t.cpu() if host else t
                return allgather_rows(src, self.group).to(t.device)
            a = {k: ag(v) for k, v in a.items()}
            lv = ag(lv.to(a["sigma"].device if not host else torch.device("cpu")))
        mesh = self.ops.make_mesh(a)
        return (mesh, lv.cpu().numpy().astype(np.int8)) if with_levels else mesh


class DeviceShardOps:
    """Per-rank device state and operations of ShardedTraversal: this rank's
    vertex / edge hash tables (csrc/traverse.cu), vertex arrays, the edge
    counts of its vertices and its boundary rays; the C-ABI calls of
    csrc/shard.cu and the native level driver."""

    def __init__(self, ns, vcap_hint=None, ecap_hint=None):
        import ctypes
        from . import _lib
        from .graph import DeviceTraversal
        from .raycast import Workspace
        self.ctypes, self._lib = ctypes, _lib
        self.ns, self.d = ns, ns.dim
        self.tr = DeviceTraversal(ns, vcap_hint=vcap_hint, ecap_hint=ecap_hint)
        self.device = self.tr.dev
        self.L = _lib.lib()
        self.ws = Workspace()
        self.vcnt = torch.empty((self.tr.vsig.shape[0], self.d + 1), dtype=torch.int32,
                                device=self.device)
        self.work = None

    def _p(self, t):
        return self._lib.ptr(t)

    def _sh(self):
        return self._lib.stream_handle()

    def as_rows(self, a, k):
        t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(a))
        return t.to(device=self.device, dtype=torch.int32).reshape(-1, k).contiguous()

    def owner_bucket(self, rows, parts):
        n, k = rows.shape
        nb = self.ctypes.c_int64(0)
        self._lib.check(self.L.vr_shard_bucket(None, n, k, parts, None, None, None,
                                               self.ctypes.byref(nb), None), "vr_shard_bucket")
        ws = self.ws.get("bucket_ws", (max(nb.value, 1),), torch.uint8, self.device)
        perm = torch.empty(n, dtype=torch.int32, device=self.device)
        counts = torch.empty(parts, dtype=torch.int64, device=self.device)
        self._lib.check(self.L.vr_shard_bucket(self._p(rows), n, k, parts, self._p(perm),
                                               self._p(counts), self._p(ws),
                                               self.ctypes.byref(nb), self._sh()),
                        "vr_shard_bucket")
        return perm, [int(c) for c in counts.tolist()]

    def gather_rows(self, rows, perm):
        n, k = perm.shape[0], rows.shape[1]
        out = torch.empty((n, k), dtype=torch.int32, device=self.device)
        self._lib.check(self.L.vr_shard_gather_rows(self._p(rows), k, self._p(perm), n,
                                                    self._p(out), self._sh()), "gather_rows")
        return out

    def scatter_rows(self, rows, perm, n):
        k = rows.shape[1]
        out = torch.empty((n, k), dtype=torch.int32, device=self.device)
        self._lib.check(self.L.vr_shard_scatter_rows(self._p(rows), k, self._p(perm), n,
                                                     self._p(out), self._sh()), "scatter_rows")
        return out

    def vertex_edges(self, rows):
        m = rows.shape[0]
        out = torch.empty((m * (self.d + 1), self.d), dtype=torch.int32, device=self.device)
        self._lib.check(self.L.vr_vertex_edges(self._p(rows), m, self.d, self._p(out),
                                               self._sh()), "vr_vertex_edges")
        return out

    def bump(self, keys):
        tr = self.tr
        n = keys.shape[0]
        tr.ensure_edges(n)
        tr.e_ub += n
        T = tr.tables()
        out = torch.empty((n, 1), dtype=torch.int32, device=self.device)
        self._lib.check(self.L.vr_trav_bump_keys(self.ctypes.byref(T), self.d, self._p(keys), n,
                                                 self._p(out), self._sh()), "vr_trav_bump_keys")
        if int(tr.overflow.item()):
            raise RuntimeError("traversal hash table overflow")
        return out

    def set_counts(self, first, vals):
        self.vcnt[first:first + vals.shape[0]] = vals

    def add_vertices(self, rows, level, tag):
        """Claim received sigma rows; store the new ones (fp64 circumcentres)
        at the next local ids.  Returns (first id, new sigma rows)."""
        from .errors import DegenerateConfiguration
        tr, d = self.tr, self.d
        n = rows.shape[0]
        first = tr.nv
        if n == 0:
            return first, rows[:0]
        tr.ensure_vertices(n)
        if self.vcnt.shape[0] < tr.vsig.shape[0]:
            grown = torch.empty((tr.vsig.shape[0], d + 1), dtype=torch.int32, device=self.device)
            grown[:self.vcnt.shape[0]] = self.vcnt
            self.vcnt = grown
        T = tr.tables()
        lvl = 0 if level is None else int(level)
        slot = torch.empty(n, dtype=torch.int64, device=self.device)
        newf = torch.empty(n, dtype=torch.int32, device=self.device)
        self._lib.check(self.L.vr_trav_claim_sigma(self.ctypes.byref(T), d, self._p(rows), n, lvl,
                                                   self._p(slot), self._p(newf), self._sh()),
                        "vr_trav_claim_sigma")
        inc = torch.cumsum(newf, 0, dtype=torch.int64)
        noff = inc - newf.to(torch.int64)
        n_new = int(inc[-1].item())
        bad = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._lib.check(self.L.vr_trav_finalize(self.ctypes.byref(T), self._p(tr.rec), d,
                                                self._p(rows), self._p(slot), self._p(newf),
                                                self._p(noff), n, first, self._p(tr.vsig),
                                                self._p(tr.vr), self._p(bad), 0, self._sh()),
                        "vr_trav_finalize")
        if int(tr.overflow.item()):
            raise RuntimeError("traversal hash table overflow")
        if int(bad.item()):
            raise DegenerateConfiguration("a vertex has an affinely dependent sigma")
        tr.nv = first + n_new
        return first, tr.vsig[first:first + n_new]

    def frontier_rays(self, f0, f1, lvl):
        """Open edges of local vertices [f0, f1) -> rays -> pruned RayCast;
        escapes become boundary rays here; returns the hit sigma' rows."""
        from .errors import DegenerateConfiguration
        ctypes, L, p, tr, d, dev = self.ctypes, self.L, self._p, self.tr, self.d, self.device
        ws = self.ws
        F = f1 - f0
        if F <= 0:
            return dict(n_rays=0, sigma=torch.empty((0, d + 1), dtype=torch.int32, device=dev))
        fs, fr, fc = tr.vsig[f0:f1], tr.vr[f0:f1], self.vcnt[f0:f1].contiguous()
        open_mask = ws.get("sh_open_mask", (F, d + 1), torch.uint8, dev)
        open_cnt = ws.get("sh_open_cnt", (F,), torch.int32, dev)
        off = ws.get("sh_open_off", (F,), torch.int64, dev)
        nb = ctypes.c_int64(0)
        nr = ctypes.c_int64(0)
        L.vr_shard_open(None, F, d, None, None, None, None, None, ctypes.byref(nb), None)
        tmp = ws.get("sh_open_tmp", (max(nb.value, 1),), torch.uint8, dev)
        self._lib.check(L.vr_shard_open(p(fc), F, d, p(open_mask), p(open_cnt), p(off),
                                        ctypes.byref(nr), p(tmp), ctypes.byref(nb), self._sh()),
                        "vr_shard_open")
        R = int(nr.value)
        if R == 0:
            return dict(n_rays=0, sigma=torch.empty((0, d + 1), dtype=torch.int32, device=dev))
        ns = self.ns
        ix, s32 = ns.prune_index(dev), ns.screen32(dev)
        rx = ws.get("sh_rx", (R, d), torch.float64, dev)
        ru = ws.get("sh_ru", (R, d), torch.float64, dev)
        reta = ws.get("sh_reta", (R, d), torch.int32, dev)
        rpar = ws.get("sh_rpar", (R,), torch.int32, dev)
        hidx = ws.get("sh_hidx", (R,), torch.int32, dev)
        ht = ws.get("sh_ht", (R,), torch.float64, dev)
        hflag = ws.get("sh_hflag", (R,), torch.uint8, dev)
        bad = ws.get("sh_bad", (2,), torch.int32, dev)
        wsb = ctypes.c_int64(0)
        self._lib.check(L.vr_trav_level_workspace(F, R, ns.n, d, ctypes.byref(wsb)),
                        "level_workspace")
        scratch = ws.get("sh_scratch", (wsb.value,), torch.uint8, dev)
        counts = np.zeros(3, dtype=np.int64)
        self._lib.check(L.vr_trav_level_rays(
            p(tr.rec), ns.n, d, tr.sqmax, ctypes.byref(s32.struct), ctypes.byref(ix.struct),
            p(fs), p(fr), F, p(open_mask), p(off), R, p(rx), p(ru), p(reta), p(rpar), p(hidx),
            p(ht), p(hflag), p(bad), p(self.work), counts.ctypes.data, p(scratch),
            scratch.numel(), self._sh()), "vr_trav_level_rays")
        n_esc, n_deg, n_bad = (int(v) for v in counts)
        if n_bad:
            raise DegenerateConfiguration("generators of a frontier vertex are affinely dependent")
        if n_deg:
            raise DegenerateConfiguration(
                f"{n_deg} edge raycasts hit a generator on the circumsphere band")
        ok = hflag == 0
        if n_esc:
            esc = (hflag == 1).to(torch.int32)
            eoff = torch.cumsum(esc, 0, dtype=torch.int64) - esc.to(torch.int64)
            tr.ensure_boundary(n_esc)
            self._lib.check(L.vr_trav_boundary(d, p(esc), p(eoff), p(rpar), p(ru), R, p(fs),
                                               tr.nb, p(tr.bsig), p(tr.bu), self._sh()),
                            "vr_trav_boundary")
            tr.nb += n_esc
        # sigma' = sorted(eta + {i}) of the hits
        sig = torch.cat([reta[ok], hidx[ok].view(-1, 1)], 1)
        sig, _ = torch.sort(sig, 1)
        return dict(n_rays=R, sigma=sig.to(torch.int32).contiguous())

    def local_arrays(self):
        tr = self.tr
        ek, ec = tr.edges()
        return dict(sigma=tr.vsig[:tr.nv], r=tr.vr[:tr.nv], edge_key=ek, edge_count=ec,
                    boundary_sigma=tr.bsig[:tr.nb], boundary_u=tr.bu[:tr.nb])

    def make_mesh(self, a):
        from .core import Mesh
        return Mesh.from_device(self.ns, a["sigma"], a["r"], a["edge_key"], a["edge_count"],
                                a["boundary_sigma"], a["boundary_u"])
