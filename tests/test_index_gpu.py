"""The native kd prune-index build (vr_build_prune_index), the screening
frame (vr_screen32_stats) and the processing-order sort (vr_ray_order),
checked against a numpy restatement of the same construction, plus the
drop-in edge cases that ride on them (empty candidate sets, MC cells with
more faces than the first-pass table)."""
import math

import numpy as np
import pytest
import torch

import paper_2405_10050_b200 as vb
from paper_2405_10050_b200.core import PRUNE_TILE
from paper_2405_10050_b200.errors import UnboundedRay
from paper_2405_10050_b200.integrate_mc import CELL_OK, CELL_OVERFLOW

pytestmark = pytest.mark.gpu


# --- numpy restatement of the index (test infrastructure) -------------------

def kd_order_np(P, tile=PRUNE_TILE):
    """Balanced kd partition: per depth, every segment of > 1 tile is sorted
    (stably) along the widest axis of its bounding box (first axis on ties)
    and split after floor(tiles / 2) whole tiles."""
    n, d = P.shape
    order = np.arange(n)
    segs = [(0, n)]
    while True:
        nxt, did = [], False
        for a, b in segs:
            if b - a <= tile:
                nxt.append((a, b))
                continue
            did = True
            X = P[order[a:b]]
            dim = int(np.argmax(X.max(0) - X.min(0)))
            o = np.argsort(X[:, dim], kind="stable")
            order[a:b] = order[a:b][o]
            nt = (b - a + tile - 1) // tile
            m = a + (nt // 2) * tile
            nxt += [(a, m), (m, b)]
        segs = nxt
        if not did:
            return order


def heap_ranges_np(nt):
    size = 1
    while size < nt:
        size *= 2
    rng = np.full((2 * size - 1, 2), -1, dtype=np.int64)
    stack = [(0, 0, nt)]
    while stack:
        i, lo, hi = stack.pop()
        rng[i] = lo, hi
        if hi - lo > 1:
            mid = lo + (hi - lo) // 2
            stack += [(2 * i + 1, lo, mid), (2 * i + 2, mid, hi)]
    return rng


def union_boxes(tbox, ranges, d):
    out = np.zeros((len(ranges), 2 * d))
    for i, (lo, hi) in enumerate(ranges):
        if lo >= 0:
            out[i, :d] = tbox[lo:hi, :d].min(0)
            out[i, d:] = tbox[lo:hi, d:].max(0)
    return out


@pytest.mark.parametrize("n,d", [(64, 2), (65, 3), (300, 4), (1000, 5), (4097, 6),
                                  (20000, 6), (9000, 8), (2500, 7)])
def test_native_index_matches_numpy_restatement(n, d):
    pts = np.random.default_rng(n + d).standard_normal((n, d)) * np.linspace(1, 3, d)
    ns = vb.NodeSet(pts)
    ix = ns.prune_index()
    torch.cuda.synchronize()
    perm = ix.perm.cpu().numpy()
    assert np.array_equal(perm, kd_order_np(pts))
    inv = ix.inv_perm.cpu().numpy()
    assert np.array_equal(inv[perm], np.arange(n))
    rec = ix.rec.cpu().numpy()
    assert np.array_equal(rec[:n, :d], pts[perm])
    assert np.all(np.isinf(rec[n:, d])) and not rec[n:, :d].any()
    nt = (n + PRUNE_TILE - 1) // PRUNE_TILE
    P = pts[perm]
    tb = np.zeros((nt, 2 * d))
    for t in range(nt):
        blk = P[t * PRUNE_TILE:(t + 1) * PRUNE_TILE]
        tb[t, :d], tb[t, d:] = blk.min(0), blk.max(0)
    assert np.array_equal(ix.tile_box.cpu().numpy(), tb)
    ranges = heap_ranges_np(nt)
    assert np.array_equal(ix.node_range.cpu().numpy(), ranges)
    nb = union_boxes(tb, ranges, d)
    assert np.array_equal(ix.node_box.cpu().numpy(), nb)
    # fp32 rows in the centred frame contain the fp64 boxes
    c = ns.screen32().center.cpu().numpy()
    b32 = ix.node_box32.cpu().numpy().astype(np.float64)
    used = ranges[:, 0] >= 0
    assert np.all(b32[used, :d] <= nb[used, :d] - c) and np.all(b32[used, d:2 * d] >= nb[used, d:] - c)
    cb = ix.node_cb32.cpu().numpy().astype(np.float64)
    assert np.all(cb[used, :d] - cb[used, d:2 * d] <= nb[used, :d] - c)
    assert np.all(cb[used, :d] + cb[used, d:2 * d] >= nb[used, d:] - c)
    t32 = ix.tile_box32.cpu().numpy().astype(np.float64)
    assert np.all(t32[:, :d] <= tb[:, :d] - c) and np.all(t32[:, d:2 * d] >= tb[:, d:] - c)
    # 32-ary levels: unions of 32^l consecutive tiles, one root
    w = ix.wide_box32.cpu().numpy().astype(np.float64)
    assert ix.wide_cnt[0] == nt and ix.wide_cnt[-1] == 1 and len(ix.wide_cnt) >= 2
    for lvl, (off, cnt) in enumerate(zip(ix.wide_off, ix.wide_cnt)):
        span = 32 ** lvl
        for j in range(0, cnt, max(1, cnt // 7)):
            lo, hi = tb[j * span:(j + 1) * span, :d].min(0), tb[j * span:(j + 1) * span, d:].max(0)
            assert np.all(w[off + j, :d] <= lo - c) and np.all(w[off + j, d:2 * d] >= hi - c)
    # screening frame of the node set
    s32 = ns.screen32()
    want_c = 0.5 * (pts.min(0) + pts.max(0))
    assert np.array_equal(s32.center.cpu().numpy(), want_c)
    assert s32.bound == np.abs(pts - want_c).max()
    assert math.isclose(s32.sqmax, ((pts - want_c) ** 2).sum(1).max(), rel_tol=1e-15)


def test_ray_order_is_the_stable_key_sort():
    from paper_2405_10050_b200.raycast import coherent_order, ray_keys, ray_order
    pts = np.random.default_rng(3).random((5000, 6))
    ns = vb.NodeSet(pts)
    ix = ns.prune_index()
    rng = np.random.default_rng(4)
    u = torch.from_numpy(rng.standard_normal((40000, 6))).cuda()
    eta = torch.from_numpy(rng.integers(0, 5000, (40000, 2)).astype(np.int32)).cuda()
    keys = ray_keys(u, eta, ix.inv_perm).cpu().numpy()
    want = np.argsort(keys, kind="stable")
    assert np.array_equal(coherent_order(ix, eta, u).cpu().numpy(), want)
    keys_mc = ray_keys(u, rays_per_cell=100).cpu().numpy()
    got = ray_order(u, rays_per_cell=100, n_base=400).cpu().numpy()
    assert np.array_equal(got, np.argsort(keys_mc, kind="stable"))


def test_index_build_launches_no_torch_sort_or_scatter():
    """The prune index is built by the library's own kernels: no at::
    sort / scatter kernels run during NodeSet.prune_index()."""
    from torch.profiler import ProfilerActivity, profile
    pts = np.random.default_rng(5).random((30000, 8))
    ns = vb.NodeSet(pts)
    ns.device_records()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ns.prune_index()
        torch.cuda.synchronize()
    names = [e.key for e in prof.key_averages()]
    bad = [k for k in names if ("at::" in k or "at_cuda" in k) and
           any(w in k.lower() for w in ("sort", "scatter", "index", "reduce"))]
    assert not bad, bad
    assert any("k_level_bbox" in k for k in names)


def test_empty_candidate_set_escapes_like_the_reference():
    pts = np.random.default_rng(6).random((50, 3))
    ns = vb.build_node_set(pts)
    q = vb.RayQuery((0,), pts[0], np.array([0.0, 0.0, 1.0]))
    assert vb.raycast_incircle(ns, q, candidates=[]) is None
    rng = np.random.default_rng(7)
    z0 = np.random.default_rng(7).standard_normal(3)
    with pytest.raises(UnboundedRay) as e:
        vb.mc_areas_only(ns, 0, 10, rng, neighbors=[])
    assert np.allclose(e.value.direction, z0 / np.linalg.norm(z0))


def test_mc_cells_overflowing_the_face_table_are_re_reduced():
    """A first-pass face table of 4 faces overflows every interior cell; the
    cells are re-reduced with a table no cell can overflow and match the
    run with a large table bitwise (unbounded face counts, like the
    reference's dict, integrate_mc.py:147-160)."""
    pts = np.random.default_rng(8).random((4000, 4))
    ns = vb.NodeSet(pts)
    cells = np.argsort(np.linalg.norm(pts - 0.5, axis=1))[:300].astype(np.int32)
    small = vb.mc_cells(ns, cells, 500, seed=3, max_faces=4)
    big = vb.mc_cells(ns, cells, 500, seed=3, max_faces=500)
    assert (small.status == CELL_OK).all() and not (small.status == CELL_OVERFLOW).any()
    assert np.array_equal(small.face_offsets, big.face_offsets)
    assert np.array_equal(small.face_j, big.face_j)
    assert np.array_equal(small.face_area, big.face_area)
    assert np.array_equal(small.volume, big.volume)


def test_mc_face_map_in_global_memory_for_huge_face_counts():
    """d = 8 cells hit hundreds of faces; a face table sized past the
    shared-memory map (max_faces 6000 -> 16k-slot map in the global
    workspace) gives the same result as the shared-memory map."""
    pts = np.random.default_rng(9).random((20000, 8))
    ns = vb.NodeSet(pts)
    cells = np.argsort(np.linalg.norm(pts - 0.5, axis=1))[:20].astype(np.int32)
    a = vb.mc_cells(ns, cells, 3000, seed=1, max_faces=1500)
    b = vb.mc_cells(ns, cells, 3000, seed=1, max_faces=6000)
    assert np.array_equal(a.face_j, b.face_j) and np.array_equal(a.face_area, b.face_area)
    assert np.array_equal(a.volume, b.volume)
    assert (np.diff(a.face_offsets) > 50).any()
