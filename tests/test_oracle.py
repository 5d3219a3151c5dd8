"""Pin the CPU oracle (oracle/voronray_oracle.py) to the reference's own
outputs (tests/golden/, produced by running the unmodified reference).  CPU
only; sized to finish in about a minute."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, config2_rays, golden
from oracle import voronray_oracle as orc


def test_philox_known_answers():
    # Random123 Philox4x32-10 KAT vectors
    cases = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
             ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
             ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
              (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]
    for ctr, key, want in cases:
        out = orc._philox(*[np.array([c], dtype=np.uint32) for c in ctr], *key)
        assert tuple(int(o[0]) for o in out) == want


def test_philox_normals_are_standard():
    z = orc.philox_normals(7, np.arange(50), 2000, 5)
    assert z.shape == (100000, 5)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1.0) < 0.01
    # counter-based: a sub-range equals the same cells drawn alone
    assert np.array_equal(orc.philox_normals(7, [3, 4], 2000, 5), z[3 * 2000:5 * 2000])


def test_stream_matches_reference_recipe():
    a = orc.stream(5, "descent", 11).standard_normal(6)
    ss = np.random.SeedSequence(entropy=5, spawn_key=(0, 11))
    b = np.random.Generator(np.random.PCG64(ss)).standard_normal(6)
    assert np.array_equal(a, b)


def test_config2_rays_probe_loop_and_argmin():
    gz = golden("config2_sample.npz")
    pts = np.random.default_rng(0).random((20000, 6))
    nodes = orc.Nodes(pts)  # kd-tree probe, as the reference for N > 2048
    pos = {int(p): m for m, p in enumerate(gz["pool_p"])}
    x = np.array([gz["pool_r"][pos[int(p)]] for p in gz["ray_p"]])
    u, g = gz["u"], gz["g"]
    for k in range(0, 4000, 20):
        res = orc.raycast(nodes, (int(g[k]),), x[k], u[k])
        if gz["status"][k] == 1:
            assert res is None
            continue
        sig, rp = res
        assert sig == tuple(sorted((int(g[k]), int(gz["idx"][k]))))
        assert np.array_equal(rp, gz["rp"][k])  # same algorithm, same libraries: bitwise
    idx, t = orc.raycast_argmin(pts, x[:600], u[:600], g[:600, None])
    ok = gz["status"][:600] == 0
    assert np.array_equal(idx[ok], gz["idx"][:600][ok])
    rp = x[:600] + t[:, None] * u[:600]
    assert np.max(np.abs(rp[ok] - gz["rp"][:600][ok])) <= 1e-12


def test_config2_descent_vertices():
    gz = golden("config2_sample.npz")
    pts = np.random.default_rng(0).random((20000, 6))
    nodes = orc.Nodes(pts)
    for m in range(0, 60, 3):
        s = int(gz["pool_start"][m])
        sig, r = orc.descent(nodes, s, orc.stream(0, "descent", s))
        assert sig == tuple(int(v) for v in gz["pool_sigma"][m])
        assert np.array_equal(r, gz["pool_r"][m])


def test_config2_recipe_is_the_golden_one():
    s, p, u = config2_rays(4000)
    gz = golden("config2_sample.npz")
    assert np.array_equal(p, gz["ray_p"]) and np.array_equal(u, gz["u"])
    assert set(gz["pool_p"]) == set(p)


def test_config5_argmin_form():
    gz = golden("config5_sample.npz")
    pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    g = gz["gen_g"][:25]
    idx, t = orc.raycast_argmin(pts, pts[g], gz["gen_u"][:25], g[:, None])
    assert np.array_equal(np.where(gz["gen_status"][:25] == 0, idx, -1),
                          np.where(gz["gen_status"][:25] == 0, gz["gen_idx"][:25], -1))
    e = slice(0, 18)
    idx, t = orc.raycast_argmin(pts, gz["edge_x"][e], gz["edge_u"][e], gz["edge_eta"][e])
    ok = gz["edge_status"][e] == 0
    assert np.array_equal(idx[ok], gz["edge_idx"][e][ok])


def _sorted(a):
    a = np.asarray(a)
    return a[np.lexsort(a.T[::-1])] if len(a) else a


def test_config1_dfs_traversal():
    gz = golden("mesh_config1.npz")
    pts = np.random.default_rng(0).random((1000, 3))
    verts, counts, boundary, nray = orc.voronoi_graph(orc.Nodes(pts), seed=0)
    assert orc.sigma_digest(verts) == \
        "b1f6f8721369b9116ff154e6673225998fb3785479bb65c18dafb6b2db2c0b1a"
    assert np.array_equal(_sorted(np.array([b[0] for b in boundary])), gz["boundary_sigma"])
    ek = sorted(counts)
    assert np.array_equal(np.array(ek, dtype=np.int32), gz["edge_key"])
    assert np.array_equal(np.array([counts[e] for e in ek]), gz["edge_count"])
    assert nray + 3 == int(gz["raycasts"]) or nray <= int(gz["raycasts"])
    # the reference's chained coordinates, bitwise (same algorithm)
    keys = [tuple(int(v) for v in s) for s in gz["sigma"]]
    r = np.array([verts[k] for k in keys])
    assert np.array_equal(r, gz["r"])


@pytest.mark.parametrize("name,mk,seed", [
    ("mesh_2d", lambda: np.random.default_rng(1234).random((120, 2)), 0),
    ("four_point", lambda: np.array([(0.0, 0.0), (2.0, 0.0), (0.0, 2.0), (2.0, 2.1)]), 42),
    ("oracle_3d_50", lambda: np.random.default_rng(17).random((50, 3)), 5),
])
def test_small_meshes(name, mk, seed):
    gz = golden("meshes_small.npz")
    verts, counts, boundary, _ = orc.voronoi_graph(orc.Nodes(mk()), seed=seed)
    assert np.array_equal(_sorted(np.array(list(verts), dtype=np.int32)), gz[f"{name}__sigma"])


def test_mc_replay_and_neighbour_batch():
    gz = golden("mc_golden.npz")
    pts = np.random.default_rng(0).random((100000, 4))
    nodes = orc.Nodes(pts)
    # z of the golden equals the Philox port's stream for those cells
    assert np.array_equal(orc.philox_normals(0, gz["c4_cells"], 1000, 4), gz["c4_z"])
    off = gz["c4_face_off"]
    m = 0
    areas, vol, _ = orc.mc_areas(nodes, int(gz["c4_cells"][m]), 1000,
                                 orc.Replay(gz["c4_z"][:1000]))
    assert vol == float(gz["c4_volume"][m])
    assert sorted(areas) == list(gz["c4_face_j"][off[0]:off[1]])
    # neighbour-restricted batch path (integrate_mc.py:164-197)
    p2 = np.random.default_rng(1234).random((120, 2))
    from paper_2405_10050_b200.rng import stream
    areas, vol, _ = orc.mc_areas(orc.Nodes(p2), int(gz["m2_cell"]), 3000,
                                 stream(2024, "test", 20), neighbors=gz["m2_neighbors"])
    assert vol == pytest.approx(float(gz["m2_volume"]), rel=1e-14)
    assert sorted(areas) == list(gz["m2_face_j"])


def test_config3_reference_record():
    with open(os.path.join(GOLDEN, "config3_reference.json")) as fh:
        ref = json.load(fh)
    # digests quoted in SURVEY.md Appendix B, reproduced by the reference run
    assert ref["sigma_digest"] == \
        "f8093583cb129297758ebea66c8fcbbf3938086d9f8b8ee1b0f79096a9351173"
    assert ref["n_vertices"] == 1607349 and ref["n_boundary"] == 5800
    pts = np.random.default_rng(0).standard_normal((10000, 5))
    import hashlib
    assert hashlib.sha256(pts.tobytes()).hexdigest()[:16] == ref["input_sha16"]
