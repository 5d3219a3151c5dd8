"""B200 Monte-Carlo parity (SURVEY.md §8(c) rule 4): with the same normals
(replayed), the device MC equals the reference's mc_areas_only -- per-face
areas and volume within 1e-12 relative, identical face sets."""
import math

import numpy as np
import pytest

from conftest import UNIT_SQUARE_POINTS, golden

pytestmark = pytest.mark.gpu

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.errors import UnboundedRay  # noqa: E402
from paper_2405_10050_b200.rng import ReplayNormals  # noqa: E402
from oracle import voronray_oracle as orc  # noqa: E402

REL = 1e-12


def _close(a, b, rel=REL):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def _cmp_areas(got, want_j, want_a, rel=REL):
    assert sorted(got) == [int(j) for j in want_j]
    for j, a in zip(want_j, want_a):
        assert _close(got[int(j)], float(a), rel), (j, got[int(j)], a)


def test_config4_cells_replayed_normals():
    gz = golden("mc_golden.npz")
    pts = np.random.default_rng(0).random((100000, 4))
    ns = vb.NodeSet(pts)
    z = gz["c4_z"]
    off = gz["c4_face_off"]
    for m, c in enumerate(gz["c4_cells"]):
        areas, vol = vb.mc_areas_only(ns, int(c), 1000, ReplayNormals(z[m * 1000:(m + 1) * 1000]))
        assert _close(vol, float(gz["c4_volume"][m]))
        _cmp_areas(areas, gz["c4_face_j"][off[m]:off[m + 1]], gz["c4_face_area"][off[m]:off[m + 1]])


def test_batched_philox_equals_replay_of_its_own_directions():
    pts = np.random.default_rng(0).random((100000, 4))
    ns = vb.NodeSet(pts)
    gz = golden("mc_golden.npz")
    cells = gz["c4_cells"]
    res = vb.mc_cells(ns, cells, 1000, seed=0)
    z = vb.mc_directions(4, cells, 1000, seed=0)
    # device Philox normals == the numpy port of the same stream (libm vs CUDA
    # log/sincos differ in the last ulp only)
    zp = orc.philox_normals(0, cells, 1000, 4)
    assert np.max(np.abs(z - zp)) <= 1e-13 * max(1.0, np.max(np.abs(zp)))
    nodes = orc.Nodes(pts)
    for m, c in enumerate(cells[:3]):
        areas, vol, _ = orc.mc_areas(nodes, int(c), 1000, orc.Replay(z[m * 1000:(m + 1) * 1000]))
        assert res.status[m] == 0
        assert _close(float(res.volume[m]), vol)
        got = res.areas(m)
        assert sorted(got) == sorted(areas)
        for j in areas:
            assert _close(got[j], areas[j])


def test_unit_square_reference_stream():
    # reference test stream (test_integrate_mc.py:63-67) drawn on the host
    gz = golden("mc_golden.npz")
    ns = vb.build_node_set(UNIT_SQUARE_POINTS)
    areas, vol, smp = vb.mc_areas_only(ns, 0, 20000, vb.rng.stream(2024, "test", 4),
                                       return_samples=True)
    assert _close(vol, float(gz["usq_volume"]), 1e-11)
    _cmp_areas(areas, gz["usq_face_j"], gz["usq_face_area"], 1e-11)
    assert np.allclose(smp, gz["usq_samples"], rtol=1e-12, atol=0)
    # the reference's statistical contract (test_integrate_mc.py:56-67)
    areas, vol = vb.mc_areas_only(ns, 0, 100_000, vb.rng.stream(2024, "test", 3))
    assert vol == pytest.approx(1.0, rel=0.01)
    assert sum(areas.values()) == pytest.approx(4.0, rel=0.015)
    assert set(areas) == {1, 2, 3, 4}


def test_neighbour_restricted_batch_path():
    gz = golden("mc_golden.npz")
    pts = np.random.default_rng(1234).random((120, 2))
    ns = vb.build_node_set(pts)
    i = int(gz["m2_cell"])
    areas, vol = vb.mc_areas_only(ns, i, 3000, vb.rng.stream(2024, "test", 20),
                                  neighbors=gz["m2_neighbors"])
    assert _close(vol, float(gz["m2_volume"]), 1e-11)
    _cmp_areas(areas, gz["m2_face_j"], gz["m2_face_area"], 1e-11)
    # full search with the same stream: same answer (test_integrate_mc.py:118-128)
    a2, v2 = vb.mc_areas_only(ns, i, 3000, vb.rng.stream(2024, "test", 20))
    assert _close(v2, vol, 1e-11)


def test_unbounded_cell_raises_with_direction():
    gz = golden("mc_golden.npz")
    ns = vb.build_node_set(UNIT_SQUARE_POINTS)
    with pytest.raises(UnboundedRay) as info:
        vb.mc_areas_only(ns, 1, 2000, vb.rng.stream(2024, "test", 8))
    assert info.value.cell == 1
    assert info.value.direction.shape == (2,)
    assert np.allclose(info.value.direction, gz["unb_dir"], rtol=0, atol=1e-15)


def test_unbiased_over_repetitions():
    ns = vb.build_node_set(UNIT_SQUARE_POINTS)
    est = np.array([vb.mc_areas_only(ns, 0, 2000, vb.rng.stream(2024, "test", 100 + k))[1]
                    for k in range(50)])
    se = est.std(ddof=1) / math.sqrt(len(est))
    assert abs(est.mean() - 1.0) <= 3 * se


def test_batched_cells_status_unbounded():
    # hull cells of a small uniform set are unbounded -> status UNBOUNDED
    pts = np.random.default_rng(3).random((400, 3))
    ns = vb.NodeSet(pts)
    res = vb.mc_cells(ns, np.arange(400), 200, seed=7)
    assert (res.status == 1).sum() > 20 and (res.status == 0).sum() > 100
    # the first escaping ray of an UNBOUNDED cell really escapes (oracle)
    zc = vb.mc_directions(3, np.nonzero(res.status == 1)[0][:5], 200, seed=7)
    for m, c in enumerate(np.nonzero(res.status == 1)[0][:5]):
        k = int(res.first_bad[c])
        y = zc[m * 200 + k] / np.linalg.norm(zc[m * 200 + k])
        want, _ = orc.raycast_argmin(pts, pts[c][None], y[None], np.array([[c]]))
        assert want[0] == -1
    ok = np.nonzero(res.status == 0)[0][:5]
    z = vb.mc_directions(3, ok, 200, seed=7)
    nodes = orc.Nodes(pts)
    for m, c in enumerate(ok):
        areas, vol, _ = orc.mc_areas(nodes, int(c), 200, orc.Replay(z[m * 200:(m + 1) * 200]))
        assert _close(float(res.volume[c]), vol)


def test_mc_pruned_equals_exhaustive():
    pts = np.random.default_rng(0).random((100000, 4))
    ns = vb.NodeSet(pts)
    cells = np.random.default_rng(9).choice(100000, 300, replace=False)
    a = vb.mc_cells(ns, cells, 500, seed=3, mode="exhaustive", want_samples=True, screen="fp64")
    for mode in ("exhaustive", "pruned"):
        for screen in ("fp64", "fp32"):
            b = vb.mc_cells(ns, cells, 500, seed=3, mode=mode, want_samples=True, screen=screen)
            for f in ("volume", "face_offsets", "face_j", "face_area", "status", "first_bad",
                      "samples"):
                assert np.array_equal(getattr(a, f), getattr(b, f), equal_nan=True), (f, mode)


def test_config4_subset_vs_exact_volumes():
    """SURVEY §8(c) rule 5: >= 95% of the 2,000 central cells within 4 SE of
    the exact (Leibniz, reference integrate_cell_poly) volume."""
    gz = golden("config4_exact.npz")
    pts = np.random.default_rng(0).random((100000, 4))
    ns = vb.NodeSet(pts)
    cells = gz["cells"]
    res = vb.mc_cells(ns, cells, 1000, seed=0, want_samples=True)
    assert (res.status == 0).all()
    surf = vb.sphere_surface_area(4)
    smp = res.samples.reshape(len(cells), 1000)
    se = surf * smp.std(axis=1, ddof=1) / (4 * np.sqrt(1000))
    dev = np.abs(res.volume - gz["volume"])
    frac = float(np.mean(dev <= 4 * se))
    assert frac >= 0.95, frac
    # unbiased in aggregate
    assert abs(np.mean((res.volume - gz["volume"]) / se)) < 0.2


def _cmp_integrals(res, gz, name, rel_area=1e-11, rel_int=1e-10):
    js = [int(j) for j in gz[f"{name}__j"]]
    assert sorted(res.area) == js
    for j, a, sv in zip(js, gz[f"{name}__area"], gz[f"{name}__surf"]):
        assert _close(res.area[j], float(a), rel_area), (name, j)
        assert _close(res.surface_integral[j], float(sv), rel_int) or abs(sv) < 1e-300, (name, j)
    assert _close(res.volume, float(gz[f"{name}__vol"][0]), rel_area)
    assert _close(res.volume_integral, float(gz[f"{name}__vol"][1]), rel_int)


def test_mc_integrate_cell_matches_reference():
    """mc_integrate_cell (integrate_mc.py:70-121) on reference RNG streams:
    built-in integrands evaluated in the kernel, a Python callable on the host."""
    from paper_2405_10050_b200.integrands import const1, make_linear, sinx2
    gz = golden("mc_integrate_golden.npz")
    ns = vb.build_node_set(UNIT_SQUARE_POINTS)
    _cmp_integrals(vb.mc_integrate_cell(ns, 0, const1, 20000, 2, vb.rng.stream(2024, "test", 3)),
                   gz, "usq_const1")
    _cmp_integrals(vb.mc_integrate_cell(ns, 0, make_linear([1.0, -2.0, 0.5]), 5000, 3,
                                        vb.rng.stream(2024, "test", 6)), gz, "usq_linear")
    pts = np.random.default_rng(1234).random((120, 2))
    n2 = vb.build_node_set(pts)
    i = int(gz["m2_cell"])
    full = vb.mc_integrate_cell(n2, i, lambda x: x[0], 2000, 2, vb.rng.stream(2024, "test", 20))
    _cmp_integrals(full, gz, "m2_x0_full")
    sig = golden("meshes_small.npz")["mesh_2d__sigma"]
    nb = np.unique(sig[(sig == i).any(axis=1)])
    rest = vb.mc_integrate_cell(n2, i, lambda x: x[0], 2000, 2, vb.rng.stream(2024, "test", 20),
                                neighbors=nb[nb != i])
    assert rest.volume == full.volume and rest.area == full.area  # bitwise, like the reference test
    p4 = np.random.default_rng(0).random((100000, 4))
    n4 = vb.NodeSet(p4)
    for c in np.argsort(np.linalg.norm(p4 - 0.5, axis=1), kind="stable")[:2]:
        _cmp_integrals(vb.mc_integrate_cell(n4, int(c), sinx2, 1000, 3,
                                            vb.rng.stream(7, "mc", int(c))), gz, f"c4_sinx2_{int(c)}")


def test_mc_integrals_cells_device_philox():
    """Batched device integrals with Philox directions and subsample
    positions equal the host-evaluated replay of the same streams."""
    from paper_2405_10050_b200.integrands import sinx2
    pts = np.random.default_rng(0).random((100000, 4))
    ns = vb.NodeSet(pts)
    cells = np.argsort(np.linalg.norm(pts - 0.5, axis=1), kind="stable")[:4]
    res = vb.mc_integrals_cells(ns, cells, 500, 2, sinx2, seed=11)
    z = vb.mc_directions(4, cells, 500, seed=11)
    u = vb.mc_uniforms(cells, 500, 2, seed=11)
    zp = orc.philox_normals(11, cells, 500, 4)
    assert np.max(np.abs(z - zp)) <= 1e-13 * np.max(np.abs(zp))

    class R:  # replay in the reference's draw order: d normals, then m uniforms per ray
        def __init__(self, z, u):
            self.z, self.u, self.k, self.s = z, u, 0, 0

        def standard_normal(self, d):
            out = self.z[self.k]
            return out

        def random(self):
            v = self.u[self.k, self.s]
            self.s += 1
            if self.s == self.u.shape[1]:
                self.s, self.k = 0, self.k + 1
            return v

    for m_, c in enumerate(cells):
        rep = vb.mc_integrate_cell(ns, int(c), lambda x: sinx2(x), 500, 2,
                                   R(z[m_ * 500:(m_ + 1) * 500], u[m_ * 500:(m_ + 1) * 500]))
        assert _close(float(res["volume"][m_]), rep.volume)
        assert _close(float(res["vol_integral"][m_]), rep.volume_integral, 1e-11)
