"""HMC post-processing on the device (csrc/hmc.cu; reference
integrate_hmc.py:21-91) against the reference's own values
(tests/golden/hmc_io_golden.npz: reference mesh JSON + reference MC areas)
and a host restatement of the reference rules for generic integrands."""
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200 import io as vio  # noqa: E402
from paper_2405_10050_b200.errors import (MissingNeighbor, UnboundedCell,  # noqa: E402
                                          UnboundedFace)
from paper_2405_10050_b200.integrands import sinx2, make_linear  # noqa: E402


def _ref_mesh():
    pts = np.random.default_rng(1234).random((120, 2))
    ns = vb.NodeSet(pts)
    return ns, vio.mesh_from_dict(vio.load_json(os.path.join(GOLDEN, "mesh_2d_reference.json")), ns)


def _host_interface(mesh, i, j, A, f):
    """integrate_hmc.py:42-64 restated on the mesh's host views (test oracle)."""
    verts = mesh.face_vertices(i, j)
    d = mesh.nodes.dim
    coords = np.array([v.r for v in verts])
    return (d * math.fsum(f(v.r) for v in verts) / len(verts) + f(coords.mean(axis=0))) * A / (d + 1)


def test_hmc_matches_reference_values():
    gz = golden("hmc_io_golden.npz")
    ns, mesh = _ref_mesh()
    for c in gz["cells"]:
        areas = {int(j): float(a) for j, a in zip(gz[f"c{c}__j"], gz[f"c{c}__area"])}
        hv = vb.hmc_volume(ns, int(c), areas, mesh)
        ci = vb.hmc_cell_integral(mesh, int(c), sinx2, areas, hv)
        assert hv == pytest.approx(gz[f"c{c}__hmc"][0], rel=1e-14)
        assert ci == pytest.approx(gz[f"c{c}__hmc"][1], rel=1e-13)
        fi = [vb.hmc_interface_integral(mesh, int(c), int(j), areas[int(j)], sinx2)
              for j in gz[f"c{c}__j"]]
        assert np.allclose(fi, gz[f"c{c}__face"], rtol=1e-13, atol=0)
        # a generic Python callable goes through the host evaluation path
        g = lambda x: x[0] * x[1] + 1.0  # noqa: E731
        for j in list(areas)[:3]:
            want = _host_interface(mesh, int(c), j, areas[j], g)
            got = vb.hmc_interface_integral(mesh, int(c), j, areas[j], g)
            assert got == pytest.approx(want, rel=1e-14)


def test_hmc_batched_equals_drop_ins():
    """hmc_cells over a device MC result equals the per-cell drop-ins."""
    pts = np.random.default_rng(5).random((400, 3))
    ns = vb.NodeSet(pts)
    mesh = vb.voronoi_graph(ns, seed=0)
    cells = np.array(mesh.bounded_cells()[:40], dtype=np.int32)
    mc = vb.mc_cells(ns, cells, 2000, seed=4)
    lin = make_linear([0.5, -1.0, 2.0, 0.25])
    res = vb.hmc_cells(mesh, mc, lin)
    for k, c in enumerate(cells):
        areas = mc.areas(k)
        try:
            hv = vb.hmc_volume(ns, int(c), areas, mesh)
        except MissingNeighbor:
            assert res.status[k] & 2
            continue
        assert res.volume[k] == pytest.approx(hv, rel=1e-15)
        ci = vb.hmc_cell_integral(mesh, int(c), lin, areas, res.volume[k])
        assert res.cell_integral[k] == pytest.approx(ci, rel=1e-13)
        # pyramid volume of the MC areas vs the MC volume: same cell
        assert res.volume[k] == pytest.approx(mc.volume[k], rel=0.2)


def test_hmc_errors_like_the_reference():
    ns, mesh = _ref_mesh()
    unb = sorted(mesh.unbounded_cells())[0]
    with pytest.raises(UnboundedCell):
        vb.hmc_cell_integral(mesh, unb, sinx2, {j: 1.0 for j in mesh.neighbors(unb)}, 1.0)
    # an unbounded interface of that cell
    j = next(j for j in mesh.neighbors(unb) if mesh.face_is_unbounded(unb, j))
    with pytest.raises(UnboundedFace, match="is unbounded"):
        vb.hmc_interface_integral(mesh, unb, j, 1.0, sinx2)
    # a pair that is not an interface: 0 vertices
    c = mesh.bounded_cells()[0]
    far = next(k for k in range(ns.n) if k != c and k not in mesh.neighbors(c))
    with pytest.raises(UnboundedFace, match="has only 0 vertices"):
        vb.hmc_interface_integral(mesh, c, far, 1.0, sinx2)
    # missing neighbour areas
    nb = list(mesh.neighbors(c))
    with pytest.raises(MissingNeighbor):
        vb.hmc_volume(ns, c, {j: 1.0 for j in nb[1:]}, mesh)
    # without a mesh no neighbour check (reference semantics)
    v = vb.hmc_volume(ns, c, {j: 1.0 for j in nb[1:]})
    want = sum(0.5 * np.linalg.norm(ns.points[j] - ns.points[c]) for j in nb[1:]) / 2
    assert v == pytest.approx(want, rel=1e-15)


def test_device_mesh_to_reference_json():
    """A GPU traversal serialised with the reference's key order: sigma rows
    and boundary sigma equal the reference mesh JSON, coordinates and ray
    directions within 1e-9 (fresh fp64 circumcentres, SURVEY §8(c) rule 3)."""
    ns, ref = _ref_mesh()
    mesh = vb.voronoi_graph(ns, seed=0)
    got = vio.mesh_to_dict(mesh)
    want = vio.load_json(os.path.join(GOLDEN, "mesh_2d_reference.json"))
    assert sorted(got) == sorted(want) and got["dim"] == 2 and got["n_nodes"] == 120
    assert [v["sigma"] for v in got["vertices"]] == [v["sigma"] for v in want["vertices"]]
    for a, b in zip(got["vertices"], want["vertices"]):
        assert np.linalg.norm(np.subtract(a["r"], b["r"])) <= 1e-9 * max(1.0, np.linalg.norm(b["r"]))
    assert [b["sigma"] for b in got["boundary_rays"]] == [b["sigma"] for b in want["boundary_rays"]]
    for a, b in zip(got["boundary_rays"], want["boundary_rays"]):
        assert np.allclose(a["u"], b["u"], atol=1e-9, rtol=0)
    rt = vio.mesh_from_dict(got, ns)
    assert rt.edge_counts == mesh.edge_counts
