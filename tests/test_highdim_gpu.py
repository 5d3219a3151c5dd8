"""d = 9 .. 16 (the reference NodeSet accepts any d >= 2, core.py:44-57):
the exhaustive fp64 RayCast, the traversal and MC take over above the d <= 8
fast paths, with the same parity bars as below -- bit-exact indices and
escapes, identical vertex sets / boundary multisets / edge counts against
the oracle's restatement of the reference DFS, MC within 1e-12 under the
same normals."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2405_10050_b200 as vb  # noqa: E402
from oracle import voronray_oracle as orc  # noqa: E402


@pytest.mark.parametrize("d", [9, 12, 16])
def test_raycast_high_d_vs_oracle(d):
    pts = np.random.default_rng(d).random((3000, d))
    ns = vb.NodeSet(pts)
    assert not ns.fast_paths and ns.screen32() is None
    rng = np.random.default_rng(d + 1)
    g = rng.integers(0, 3000, 4000).astype(np.int32)
    u = rng.standard_normal((4000, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    idx, t, rp, flag = vb.raycast_batch(ns, pts[g], u, g[:, None]).to_host()
    want_idx, want_t = orc.raycast_argmin(pts, pts[g], u, g[:, None])
    assert np.array_equal(idx, want_idx)
    ok = want_idx >= 0
    assert np.allclose(t[ok], want_t[ok], rtol=1e-12, atol=0)
    assert (flag[~ok] == 1).all()
    # drop-in single ray
    res = vb.raycast_incircle(ns, vb.RayQuery((int(g[0]),), pts[g[0]], u[0]))
    if want_idx[0] < 0:
        assert res is None
    else:
        assert res[0] == tuple(sorted((int(g[0]), int(want_idx[0]))))


@pytest.mark.parametrize("n,d", [(22, 9), (24, 10)])
def test_full_diagram_high_d_vs_oracle_dfs(n, d):
    pts = np.random.default_rng(d).random((n, d))
    verts, counts, boundary, _ = orc.voronoi_graph(orc.Nodes(pts), seed=0)
    mesh = vb.voronoi_graph(vb.build_node_set(pts), seed=0)
    a = mesh.arrays()
    assert {tuple(r) for r in a["sigma"].tolist()} == set(verts)
    assert sorted(tuple(r) for r in a["boundary_sigma"].tolist()) == sorted(s for s, _ in boundary)
    assert {tuple(k): int(c) for k, c in zip(a["edge_key"].tolist(), a["edge_count"].tolist())} \
        == counts
    for k in range(0, len(a["sigma"]), 97):
        want = orc.circumcenter(pts, a["sigma"][k])
        assert np.linalg.norm(a["r"][k] - want) <= 1e-9 * max(1.0, np.linalg.norm(want))
    assert vb.verify_mesh(mesh, oracle=False).passed


def test_mc_high_d_replayed_normals_vs_oracle():
    d = 9
    pts = np.random.default_rng(3).standard_normal((3000, d))
    ns = vb.NodeSet(pts)
    cell = int(np.argmin(np.linalg.norm(pts, axis=1)))
    z = np.random.default_rng(4).standard_normal((300, d))
    areas, vol = vb.mc_areas_only(ns, cell, 300, vb.rng.ReplayNormals(z))
    a2, v2, _ = orc.mc_areas(orc.Nodes(pts), cell, 300, orc.Replay(z))
    assert sorted(areas) == sorted(a2)
    assert abs(vol - v2) <= 1e-12 * abs(v2)
    for j in areas:
        assert abs(areas[j] - a2[j]) <= 1e-12 * abs(a2[j])


def test_descent_high_d_matches_oracle():
    d = 12
    pts = np.random.default_rng(5).random((2000, d))
    ns = vb.NodeSet(pts)
    starts = [3, 77, 1500]
    sig, r = vb.descent_batch(ns, starts, seed=0)
    nodes = orc.Nodes(pts)
    for k, s in enumerate(starts):
        want, _ = orc.descent(nodes, s, orc.stream(0, "descent", s))
        assert tuple(sig[k]) == tuple(want)
