"""Multi-rank host logic on CPU (gloo, world_size 2): sharding, variable-
length all-gather, the per-level sharded RayCast exchange of the traversal
(driven here by the CPU oracle as the per-rank raycaster), MC gathers."""
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from conftest import golden
from paper_2405_10050_b200 import parallel
from oracle import voronray_oracle as orc


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, size, port, fn, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=size)
    try:
        q.put((rank, fn(rank, size)))
    finally:
        dist.destroy_process_group()


def spawn(fn, size=2):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_run, args=(r, size, port, fn, q)) for r in range(size)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(size))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(size)]


def test_shard_bounds_cover_exactly():
    for n in (0, 1, 7, 100, 1001):
        for size in (1, 2, 3, 8):
            spans = [parallel.shard_bounds(n, size, r) for r in range(size)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _allgather(rank, size):
    t = torch.arange(rank * 10, rank * 10 + 3 + rank, dtype=torch.int64).view(-1, 1)
    return parallel.allgather_rows(t).view(-1).tolist()


def test_allgather_rows_variable_lengths():
    outs = spawn(_allgather)
    assert outs[0] == outs[1] == [0, 1, 2, 10, 11, 12, 13]


PTS = np.random.default_rng(0).random((1000, 3))


def _oracle_fn(x, u, eta):
    idx, _ = orc.raycast_argmin(PTS, x.numpy(), u.numpy(), eta.numpy())
    flag = (idx < 0).astype(np.uint8)
    return torch.from_numpy(idx.astype(np.int32)), torch.from_numpy(flag)


def _level_bfs(rank, size):
    """Level-synchronous BFS of config 1 where every level's edge rays are
    split across the ranks by ShardedRaycast and the hits all-gathered; each
    rank applies the same deterministic claims to its replica."""
    rc = parallel.ShardedRaycast(_oracle_fn)
    nodes = orc.Nodes(PTS)
    s0, _ = orc.descent(nodes, 0, orc.stream(0, "descent", 0))
    verts, counts, boundary = {s0: 0}, {}, []
    for k in range(4):
        e = s0[:k] + s0[k + 1:]
        counts[e] = counts.get(e, 0) + 1
    frontier = [s0]
    while frontier:
        rays = []
        for s in frontier:
            r = orc.circumcenter(PTS, s)
            open_ks = [k for k in range(4) if counts.get(s[:k] + s[k + 1:], 0) < 2]
            if not open_ks:
                continue
            dirs = orc.vertex_directions(PTS, s, open_ks)
            rays += [(s, k, r, dirs[k]) for k in open_ks]
        if not rays:
            break
        x = torch.tensor(np.array([r[2] for r in rays]))
        u = torch.tensor(np.array([r[3] for r in rays]))
        eta = torch.tensor(np.array([s[:k] + s[k + 1:] for s, k, _, _ in rays], dtype=np.int32))
        idx, flag = rc(x, u, eta)
        nxt = []
        for (s, k, _, uu), i, f in zip(rays, idx.tolist(), flag.tolist()):
            if f == 1:
                boundary.append(s)
                continue
            new = tuple(sorted(s[:k] + s[k + 1:] + (i,)))
            if new not in verts:
                verts[new] = len(verts)
                nxt.append(new)
        for s in nxt:
            for k in range(4):
                e = s[:k] + s[k + 1:]
                counts[e] = counts.get(e, 0) + 1
        frontier = nxt
    return orc.sigma_digest(verts), sorted(boundary), len(counts)


def test_sharded_level_exchange_reproduces_config1():
    gz = golden("mesh_config1.npz")
    outs = spawn(_level_bfs)
    assert outs[0] == outs[1]
    dig, bnd, ne = outs[0]
    assert dig == "b1f6f8721369b9116ff154e6673225998fb3785479bb65c18dafb6b2db2c0b1a"
    assert np.array_equal(np.array(bnd, dtype=np.int32), gz["boundary_sigma"])
    assert ne == len(gz["edge_key"])


def _mc_gather(rank, size):
    from paper_2405_10050_b200.integrate_mc import MCResult
    rng = np.random.default_rng(rank)
    nc = 3 + rank
    nf = rng.integers(1, 5, nc)
    off = np.concatenate([[0], np.cumsum(nf)])
    part = MCResult(cells=np.arange(nc) + 100 * rank, volume=rng.random(nc), face_offsets=off,
                    face_j=rng.integers(0, 50, off[-1]).astype(np.int32),
                    face_area=rng.random(off[-1]), status=np.zeros(nc, dtype=np.int32),
                    first_bad=np.full(nc, -1), samples=None)
    g = parallel.gather_mc(part, device=torch.device("cpu"))
    return (g.cells.tolist(), g.volume.tolist(), g.face_offsets.tolist(), g.face_j.tolist(),
            [part.cells.tolist(), part.volume.tolist()])


def test_gather_mc_concatenates_in_rank_order():
    outs = spawn(_mc_gather)
    assert outs[0][:4] == outs[1][:4]
    cells, vol, off, fj, _ = outs[0]
    assert cells == outs[0][4][0] + outs[1][4][0]
    assert vol == outs[0][4][1] + outs[1][4][1]
    assert off[0] == 0 and off[-1] == len(fj)


class HostShardOps:
    """Test double of parallel.DeviceShardOps on the host: the same per-rank
    operations over Python dicts, with the oracle's closed-form RayCast.  It
    drives parallel.ShardedTraversal's level protocol (owner-sharded vertex
    and edge tables, all-to-all of hit sigmas and of edge keys with the
    counts replied) on CPU ranks; the product path runs DeviceShardOps."""

    device = torch.device("cpu")

    def __init__(self, pts):
        self.p, self.d = pts, pts.shape[1]
        self.vid, self.sig, self.r, self.cnt = {}, [], [], []
        self.ecount = {}
        self.bsig, self.bu = [], []

    def as_rows(self, a, k):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.int32).reshape(-1, k)

    @staticmethod
    def _owner(row, parts):
        h = 0
        for x in row:
            h = (h * 1000003 + int(x)) & 0xFFFFFFFF
        return (h ^ (h >> 13)) % parts

    def owner_bucket(self, rows, parts):
        own = np.array([self._owner(r, parts) for r in rows.tolist()], dtype=np.int64)
        perm = np.argsort(own, kind="stable")
        counts = np.bincount(own, minlength=parts)
        return torch.as_tensor(perm.astype(np.int64)), [int(c) for c in counts]

    def gather_rows(self, rows, perm):
        return rows[perm].contiguous()

    def scatter_rows(self, rows, perm, n):
        out = torch.empty((n, rows.shape[1]), dtype=torch.int32)
        out[perm] = rows.to(torch.int32)
        return out

    def vertex_edges(self, rows):
        d1 = self.d + 1
        out = [r[:k] + r[k + 1:] for r in rows.tolist() for k in range(d1)]
        return torch.tensor(out, dtype=torch.int32).reshape(-1, self.d)

    def bump(self, keys):
        ks = [tuple(k) for k in keys.tolist()]
        for k in ks:
            self.ecount[k] = self.ecount.get(k, 0) + 1
        return torch.tensor([[self.ecount[k]] for k in ks], dtype=torch.int32).reshape(-1, 1)

    def set_counts(self, first, vals):
        for i, row in enumerate(vals.tolist()):
            self.cnt[first + i] = row

    def add_vertices(self, rows, level, tag):
        first = len(self.sig)
        new = []
        for row in rows.tolist():
            t = tuple(row)
            if t not in self.vid:
                self.vid[t] = len(self.sig)
                self.sig.append(t)
                self.r.append(orc.circumcenter(self.p, t))
                self.cnt.append([0] * (self.d + 1))
                new.append(t)
        return first, torch.tensor(new, dtype=torch.int32).reshape(-1, self.d + 1)

    def frontier_rays(self, f0, f1, lvl):
        d = self.d
        rays = []
        for v in range(f0, f1):
            s = self.sig[v]
            open_ks = [k for k in range(d + 1) if self.cnt[v][k] < 2]
            if open_ks:
                dirs = orc.vertex_directions(self.p, s, open_ks)
                rays += [(s, k, self.r[v], dirs[k]) for k in open_ks]
        if not rays:
            return dict(n_rays=0, sigma=torch.zeros((0, d + 1), dtype=torch.int32))
        x = np.array([r[2] for r in rays])
        u = np.array([r[3] for r in rays])
        eta = np.array([s[:k] + s[k + 1:] for s, k, _, _ in rays], dtype=np.int32)
        idx, _ = orc.raycast_argmin(self.p, x, u, eta)
        out = []
        for (s, k, _, uu), i in zip(rays, idx.tolist()):
            if i < 0:
                self.bsig.append(s)
                self.bu.append(uu)
            else:
                out.append(sorted(s[:k] + s[k + 1:] + (i,)))
        return dict(n_rays=len(rays), sigma=torch.tensor(out, dtype=torch.int32).reshape(-1, d + 1))

    def local_arrays(self):
        d = self.d
        ek = list(self.ecount)
        return dict(sigma=torch.tensor(self.sig, dtype=torch.int32).reshape(-1, d + 1),
                    r=torch.tensor(np.array(self.r)).reshape(-1, d),
                    edge_key=torch.tensor(ek, dtype=torch.int32).reshape(-1, d),
                    edge_count=torch.tensor([self.ecount[k] for k in ek], dtype=torch.int32),
                    boundary_sigma=torch.tensor(self.bsig, dtype=torch.int32).reshape(-1, d + 1),
                    boundary_u=torch.tensor(np.array(self.bu)).reshape(-1, d))

    def make_mesh(self, a):
        return {k: v.numpy() for k, v in a.items()}


def _owner_sharded(rank, size):
    """Config 1 through parallel.ShardedTraversal: each rank owns a hash
    shard of the vertices and edges and raycasts its own frontier."""
    from paper_2405_10050_b200 import NodeSet
    ns = NodeSet(PTS)
    nodes = orc.Nodes(PTS)
    s0, _ = orc.descent(nodes, 0, orc.stream(0, "descent", 0))
    st = parallel.ShardedTraversal(ns, HostShardOps(PTS))
    st.seed(np.array([s0], dtype=np.int32))
    lvl, per_level = 1, []
    while True:
        n = st.level(lvl)
        per_level.append(n)
        if n == 0:
            break
        lvl += 1
    own_v = len(st.ops.sig)
    a, lv = st.gather(with_levels=True)
    sig = a["sigma"]
    return (orc.sigma_digest([tuple(r) for r in sig.tolist()]),
            sorted(tuple(r) for r in a["boundary_sigma"].tolist()),
            sorted((tuple(k), int(c)) for k, c in zip(a["edge_key"].tolist(),
                                                     a["edge_count"].tolist())),
            own_v, per_level, st.rays)


def test_owner_sharded_traversal_reproduces_config1():
    """Two ranks with owner-sharded tables (hash(sigma) / hash(eta) mod 2,
    per-level all-to-all of hit sigmas and edge keys, counts replied)
    reproduce the reference's config-1 vertex set, boundary multiset and
    edge counts; both ranks own a real share of the vertices."""
    gz = golden("mesh_config1.npz")
    outs = spawn(_owner_sharded)
    assert outs[0][:3] == outs[1][:3]
    three = spawn(_owner_sharded, size=3)  # an odd rank count partitions differently
    assert three[0][:3] == three[2][:3] == outs[0][:3]
    dig, bnd, edges, _, levels, _ = outs[0]
    assert dig == "b1f6f8721369b9116ff154e6673225998fb3785479bb65c18dafb6b2db2c0b1a"
    assert np.array_equal(np.array(bnd, dtype=np.int32), gz["boundary_sigma"])
    want = sorted((tuple(k), int(c)) for k, c in zip(gz["edge_key"].tolist(),
                                                     gz["edge_count"].tolist()))
    assert edges == want
    assert sum(levels) + 1 == 6341
    shares = [o[3] for o in outs]
    assert sum(shares) == 6341 and min(shares) > 6341 // 4
    assert outs[0][5] + outs[1][5] > 0
