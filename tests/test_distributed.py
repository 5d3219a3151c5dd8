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
