"""Multi-GPU sharding: one process per GPU, torch.distributed
(NCCL over NVLink on B200 boxes, gloo for CPU tests) for the plumbing.

* Batched RayCast / MC: rays and cells are independent units.  Each rank
  takes a contiguous shard, generators are replicated, nothing crosses the
  link on the data path; results are gathered once at the end.  MC
  directions are keyed by (seed, cell, ray), so the answer does not depend on
  the number of ranks.
* Traversal: the vertex / edge tables are replicated; the open edges of each
  level (identical on every rank, since the replicas are identical) are split
  across ranks, every rank raycasts its slice, and one all-gather per level
  exchanges the hit index + flag of every ray (5 bytes per ray).  Every rank
  then applies the same deterministic claim / finalize step, so the replicas
  stay identical.  The raycasts -- the dominant cost -- are sharded; the
  HBM-bound table updates are cheap enough to replicate (config 5 at L=5 is
  ~10 GB of tables per GPU against 180 GB of HBM).
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
