"""B200 RayCast parity: CUDA path (through the C-ABI) vs the reference's
golden vectors and the CPU oracle.  Bar: bit-exact generator indices and
escape status; coordinates within 1e-9 * max(1, |r'|)."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.errors import DegenerateConfiguration  # noqa: E402
from oracle import voronray_oracle as orc  # noqa: E402

COORD_TOL = 1e-9


def _arr(*xs):
    return np.asarray(xs, dtype=float)


def triangle_ns():
    return vb.build_node_set([(0.0, 0.0), (1.0, 0.0), (0.0, 1.0)])


def test_triangle_finds_circumcenter():
    # reference test_raycast.py:102-110
    stats = vb.RaycastStats()
    res = vb.raycast_incircle(triangle_ns(), vb.RayQuery((0, 1), _arr(0.5, 0.0), _arr(0.0, 1.0)), stats)
    sigma, rp = res
    assert sigma == (0, 1, 2)
    assert np.allclose(rp, [0.5, 0.5], atol=1e-12)
    assert stats.nn_calls >= 1 and stats.raycasts == 1


def test_triangle_escapes_downward():
    # test_raycast.py:113-116
    assert vb.raycast_incircle(triangle_ns(), vb.RayQuery((0, 1), _arr(0.5, 0.0), _arr(0.0, -1.0))) is None


def test_cocircular_square_raises_degenerate():
    # test_raycast.py:145-148: exact tie -> recheck -> runner-up band
    ns = vb.build_node_set([(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (0.0, 1.0)])
    with pytest.raises(DegenerateConfiguration):
        vb.raycast_incircle(ns, vb.RayQuery((0, 1), _arr(0.5, 0.0), _arr(0.0, 1.0)))


def test_near_degenerate_goes_through_recheck():
    # a fifth point 1e-13 outside the square's circumcircle: the screening
    # band flags the ray, the exact pass applies the reference band test
    c = np.array([0.5, 0.5])
    rad = np.sqrt(0.5)
    p5 = c + (rad * (1 + 1e-13)) * np.array([np.cos(1.0), np.sin(1.0)])
    ns = vb.build_node_set([(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), tuple(p5)])
    with pytest.raises(DegenerateConfiguration):
        vb.raycast_incircle(ns, vb.RayQuery((0, 1), _arr(0.5, 0.0), _arr(0.0, 1.0)))
    # moved well outside the band: a regular hit
    p5 = c + (rad * 1.01) * np.array([np.cos(1.0), np.sin(1.0)])
    ns = vb.build_node_set([(0.0, 0.0), (1.0, 0.0), (1.0, 1.0), tuple(p5)])
    sigma, rp = vb.raycast_incircle(ns, vb.RayQuery((0, 1), _arr(0.5, 0.0), _arr(0.0, 1.0)))
    assert sigma == (0, 1, 2)


def _check_against(ns, x, u, eta, status, idx, rp):
    res = vb.raycast_batch(ns, x, u, eta)
    gi, gt, grp, gf = res.to_host()
    ok = status == 0
    assert np.array_equal(gf[status == 1], np.ones(int((status == 1).sum()), dtype=np.uint8))
    assert np.array_equal(gi[ok], idx[ok])
    scale = np.maximum(1.0, np.linalg.norm(rp[ok], axis=1))
    err = np.linalg.norm(grp[ok] - rp[ok], axis=1) / scale
    assert err.max(initial=0.0) <= COORD_TOL, err.max()
    assert np.all(gf[ok] == 0)
    return gi, grp, gf


def test_config2_golden_rays():
    """First 4000 canonical config-2 rays vs the unmodified reference."""
    gz = golden("config2_sample.npz")
    pts = np.random.default_rng(0).random((20000, 6))
    ns = vb.build_node_set(pts)
    pos = {int(p): m for m, p in enumerate(gz["pool_p"])}
    x = np.array([gz["pool_r"][pos[int(p)]] for p in gz["ray_p"]])
    _check_against(ns, x, gz["u"], gz["g"][:, None], gz["status"], gz["idx"], gz["rp"])


def test_config2_descent_vertices_match_reference():
    gz = golden("config2_sample.npz")
    pts = np.random.default_rng(0).random((20000, 6))
    ns = vb.build_node_set(pts)
    starts = gz["pool_start"][:300]
    sig, r = vb.descent_batch(ns, starts, seed=0)
    assert np.array_equal(sig, gz["pool_sigma"][:300])
    err = np.linalg.norm(r - gz["pool_r"][:300], axis=1) / np.maximum(1, np.linalg.norm(r, axis=1))
    assert err.max() <= COORD_TOL
    # single-start drop-in agrees with the batched form
    v = vb.descent(ns, int(starts[0]), vb.rng.stream(0, "descent", int(starts[0])))
    assert v.sigma == tuple(int(s) for s in gz["pool_sigma"][0])


def test_config5_golden_rays():
    """N=1e6, d=8 (fp32-upcast generators): generator-start and edge rays."""
    gz = golden("config5_sample.npz")
    pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    ns = vb.NodeSet(pts)
    g = gz["gen_g"]
    _check_against(ns, pts[g], gz["gen_u"], g[:, None], gz["gen_status"], gz["gen_idx"], gz["gen_rp"])
    _check_against(ns, gz["edge_x"], gz["edge_u"], gz["edge_eta"], gz["edge_status"],
                   gz["edge_idx"], gz["edge_rp"])


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6, 7, 8])
def test_random_rays_vs_oracle_all_dims(d):
    rng = np.random.default_rng(100 + d)
    n = 3000 if d <= 5 else 6000
    pts = rng.random((n, d))
    ns = vb.build_node_set(pts)
    m = 700
    g = rng.integers(0, n, m)
    u = rng.standard_normal((m, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    want_idx, want_t = orc.raycast_argmin(pts, pts[g], u, g[:, None])
    res = vb.raycast_batch(ns, pts[g], u, g[:, None])
    gi, gt, grp, gf = res.to_host()
    assert np.array_equal(gi, np.where(want_idx >= 0, want_idx, -1))
    assert np.array_equal(gf == 1, want_idx < 0)
    ok = want_idx >= 0
    assert np.allclose(gt[ok], want_t[ok], rtol=1e-12, atol=0)
    # iterative probe loop (the reference algorithm itself) on a subset
    nodes = orc.Nodes(pts)
    for k in range(0, m, 35):
        r = orc.raycast(nodes, (int(g[k]),), pts[g[k]], u[k])
        if r is None:
            assert gi[k] == -1
        else:
            assert tuple(sorted((int(g[k]), int(gi[k])))) == r[0]
            assert np.linalg.norm(grp[k] - r[1]) <= COORD_TOL * max(1, np.linalg.norm(r[1]))


def test_candidate_restriction_matches_full_search():
    # reference test_raycast.py:151-164 on a cell's Voronoi neighbours
    gz = golden("meshes_small.npz")
    pts = np.random.default_rng(1234).random((120, 2))
    ns = vb.build_node_set(pts)
    sig = gz["mesh_2d__sigma"]
    i = 57
    nb = np.unique(sig[(sig == i).any(axis=1)])
    nb = nb[nb != i]
    rng = np.random.default_rng(0)
    y = rng.standard_normal((50, 2))
    y /= np.linalg.norm(y, axis=1, keepdims=True)
    full = vb.raycast_batch(ns, np.repeat(pts[i:i + 1], 50, 0), y, np.full((50, 1), i)).to_host()
    rest = vb.raycast_batch(ns, np.repeat(pts[i:i + 1], 50, 0), y, np.full((50, 1), i),
                            candidates=nb).to_host()
    assert np.array_equal(full[0], rest[0])
    assert np.array_equal(full[2], rest[2])


def test_edge_cases_sizes():
    ns = vb.build_node_set([(0.0, 0.0), (1.0, 0.0), (0.0, 1.0)])
    # zero rays
    res = vb.raycast_batch(ns, np.zeros((0, 2)), np.zeros((0, 2)), np.zeros((0, 1), dtype=np.int32))
    assert res.idx.shape[0] == 0
    # rays not a multiple of the CTA ray block, N = d + 1
    rng = np.random.default_rng(5)
    u = rng.standard_normal((1000, 2))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    gi, _, _, gf = vb.raycast_batch(ns, np.zeros((1000, 2)), u, np.zeros((1000, 1), dtype=np.int32)).to_host()
    want, _ = orc.raycast_argmin(ns.points, np.zeros((1000, 2)), u, np.zeros((1000, 1), dtype=int))
    assert np.array_equal(gi, want)


def test_vertex_directions_match_reference_helper():
    gz = golden("meshes_small.npz")
    pts = np.random.default_rng(999).random((90, 3))
    ns = vb.build_node_set(pts)
    sig = gz["mesh_3d__sigma"][:40]
    u, ok = vb.vertex_directions_batch(ns, sig)
    u = u.cpu().numpy()
    assert ok.cpu().numpy().all()
    for v in range(len(sig)):
        want = orc.vertex_directions(pts, tuple(sig[v]), range(4))
        for k in range(4):
            assert float(u[v, k] @ want[k]) >= 1.0 - 1e-12


def test_nearest_and_verify():
    rng = np.random.default_rng(7)
    pts = rng.random((60, 3))
    ns = vb.NodeSet(pts)
    q = rng.random(3)
    skip = lambda i: i % 3 == 0  # noqa: E731
    (i1, d1), d2 = ns.nearest2(q, skip)
    dists = sorted((float(np.linalg.norm(p - q)), i) for i, p in enumerate(pts) if i % 3 != 0)
    assert i1 == dists[0][1]
    assert d1 == pytest.approx(dists[0][0])
    assert d2 == pytest.approx(dists[1][0])
    assert vb.nearest_neighbor(ns, q, skip=lambda i: True) is None
    tie = vb.NodeSet([(1.0, 0.0), (-1.0, 0.0), (0.0, 3.0)])
    assert tie.nearest(np.zeros(2))[0] == 0


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6, 7, 8])
def test_pruned_equals_exhaustive(d):
    """The kd-tile pruning certificate never changes a result (bitwise)."""
    rng = np.random.default_rng(300 + d)
    n = 20000 if d <= 6 else 50000
    pts = rng.random((n, d)) if d % 2 else rng.standard_normal((n, d))
    ns = vb.build_node_set(pts)
    m = 20000
    g = rng.integers(0, n, m)
    u = rng.standard_normal((m, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    a = vb.raycast_batch(ns, pts[g], u, g[:, None], mode="exhaustive", screen="fp64").to_host()
    for mode in ("exhaustive", "pruned"):
        for screen in ("fp64", "fp32"):
            b = vb.raycast_batch(ns, pts[g], u, g[:, None], mode=mode, screen=screen).to_host()
            for x, y in zip(a, b):
                assert np.array_equal(x, y, equal_nan=True), (mode, screen)
    # edge rays with |eta| = d from descent vertices
    sig, r = vb.descent_batch(ns, rng.choice(n, 200, replace=False), seed=1)
    uu, ok = vb.vertex_directions_batch(ns, sig)
    uu = uu.cpu().numpy().reshape(-1, d)
    xs = np.repeat(r, d + 1, axis=0)
    eta = np.array([[s[j] for j in range(d + 1) if j != k] for s in sig for k in range(d + 1)])
    a = vb.raycast_batch(ns, xs, uu, eta, mode="exhaustive", screen="fp64").to_host()
    for mode in ("exhaustive", "pruned"):
        for screen in ("fp64", "fp32"):
            b = vb.raycast_batch(ns, xs, uu, eta, mode=mode, screen=screen).to_host()
            for x, y in zip(a, b):
                assert np.array_equal(x, y, equal_nan=True), (mode, screen)


@pytest.mark.gpu
@pytest.mark.parametrize("d", [5, 6])
def test_sweep_kernel_matches_exhaustive(d, monkeypatch):
    """The opt-in sweeps -- tcgen05 (VR_SWEEP=1: every generator screened by
    one M=128 x N=128 tf32 MMA per step, TMEM double-buffered) and mma.sync
    (VR_HSWEEP=1: 128-ray CTAs over a TMA ring of 256-candidate blocks) --
    are bitwise equal to the exhaustive fp64 kernel on generator-start and
    edge rays, including whatever rays start without a seed sphere."""
    import torch
    rng = np.random.default_rng(900 + d)
    n = 6000
    pts = rng.random((n, d)) if d % 2 else rng.standard_normal((n, d))
    ns = vb.build_node_set(pts)
    m = 5000
    g = rng.integers(0, n, m)
    u = rng.standard_normal((m, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    sig, r = vb.descent_batch(ns, rng.choice(n, 100, replace=False), seed=2)
    uu, ok = vb.vertex_directions_batch(ns, sig)
    uu = uu.cpu().numpy().reshape(-1, d)
    xs = np.repeat(r, d + 1, axis=0)
    eta = np.array([[s[j] for j in range(d + 1) if j != k] for s in sig for k in range(d + 1)])
    cases = ((pts[g], u, g[:, None]), (xs, uu, eta))
    refs = [vb.raycast_batch(ns, *c, mode="exhaustive", screen="fp64").to_host() for c in cases]
    rows = vb._lib.record_rows(n)
    # the tcgen05 sweep (VR_SWEEP) and the mma.sync sweep (VR_HSWEEP)
    for var in ("VR_SWEEP", "VR_HSWEEP"):
        monkeypatch.setenv(var, "1")
        work = torch.zeros(16, dtype=torch.int64, device="cuda")
        for c, a in zip(cases, refs):
            b = vb.raycast_batch(ns, *c, mode="pruned", work=work).to_host()
            for x, y in zip(a, b):
                assert np.array_equal(x, y, equal_nan=True), var
        # the sweep screened every record row for every ray
        assert int(work[0]) == rows * (m + len(xs)), var
        monkeypatch.delenv(var)


_COOP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2405_10050_b200 as vb
bad = 0
for n, d, seed in ((6000, 8, 0), (5000, 6, 1), (3000, 4, 2)):
    pts = np.random.default_rng(seed).random((n, d))
    ns = vb.NodeSet(pts)
    sig, r = vb.descent_batch(ns, np.arange(0, n, n // 40), seed=0)
    u, ok = vb.vertex_directions_batch(ns, sig)
    u = u.cpu().numpy().reshape(-1, d)
    x = np.repeat(r, d + 1, axis=0)
    eta = np.stack([np.delete(s_, k) for s_ in sig for k in range(d + 1)]).astype(np.int32)
    eta.sort(axis=1)
    rng = np.random.default_rng(seed + 10)
    g = rng.integers(0, n, 2000).astype(np.int32)
    ug = rng.standard_normal((2000, d))
    ug /= np.linalg.norm(ug, axis=1, keepdims=True)
    for xx, uu, ee in ((x, u, eta), (pts[g], ug, g[:, None])):
        a = vb.raycast_batch(ns, xx, uu, ee, mode="pruned")
        b = vb.raycast_batch(ns, xx, uu, ee, mode="exhaustive")
        bad += int(((a.idx != b.idx) | (a.flag != b.flag)).sum().item())
        bad += int((a.t != b.t).sum().item())
print("BAD", bad)
"""


def test_coop_kernel_matches_exhaustive():
    """The opt-in cooperative warp-per-ray pruned kernel (VR_COOP=1, read once
    per process, hence the subprocess) is bitwise equal to the exhaustive
    kernel on edge rays (|eta| = d) and generator-start rays."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VR_COOP="1")
    res = subprocess.run([sys.executable, "-c", _COOP_SCRIPT, root], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "BAD 0" in res.stdout, res.stdout[-2000:]


def test_host_raycaster_pipeline_matches_device_batch():
    """The host-array pipeline (chunks over several buffers / streams, CUDA
    graph replays after the first use of each chunk shape) returns exactly
    the device batch's results, for sizes that exercise the fill / drain
    chunk schedule and a ragged tail, and on repeated runs (graph replays)."""
    import torch
    from paper_2405_10050_b200.raycast import HostRaycaster
    pts = np.random.default_rng(7).random((5000, 5))
    ns = vb.NodeSet(pts)
    rng = np.random.default_rng(8)
    for n, chunk, minc in ((70001, 1 << 14, 1 << 12), (9000, 1 << 17, 1 << 16), (1, 64, 16)):
        g = rng.integers(0, 5000, n).astype(np.int32)
        u = rng.standard_normal((n, 5))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        ref = vb.raycast_batch(ns, pts[g], u, g[:, None])
        hr = HostRaycaster(ns, n, 1, chunk=chunk, min_chunk=minc, nbuf=4, compute_streams=2)
        P = HostRaycaster.pinned
        hx, hu, hg = P((n, 5), torch.float64), P((n, 5), torch.float64), P((n, 1), torch.int32)
        hx.copy_(torch.from_numpy(pts[g]))
        hu.copy_(torch.from_numpy(u))
        hg.copy_(torch.from_numpy(g[:, None].copy()))
        hidx, ht = P((n,), torch.int32), P((n,), torch.float64)
        hrp, hfl = P((n, 5), torch.float64), P((n,), torch.uint8)
        for _ in range(3):
            hidx.fill_(-7)
            hr.run(hx, hu, hg, hidx, ht, hrp, hfl)
            assert np.array_equal(hidx.numpy(), ref.idx.cpu().numpy())
            assert np.array_equal(hfl.numpy(), ref.flag.cpu().numpy())
            assert np.array_equal(ht.numpy(), ref.t.cpu().numpy())
            assert np.array_equal(hrp.numpy(), ref.rp.cpu().numpy(), equal_nan=True)


def test_ray_keys_match_torch_restatement():
    """vr_ray_keys (processing-order keys) equals the torch formula
    inv_perm[eta0] * 256 + direction_bucket(u), and the MC form k // per."""
    import torch
    from paper_2405_10050_b200.raycast import direction_bucket, ray_keys
    pts = np.random.default_rng(11).random((3000, 7))
    ns = vb.NodeSet(pts)
    ix = ns.prune_index()
    rng = np.random.default_rng(12)
    u = torch.from_numpy(rng.standard_normal((5000, 7))).cuda()
    u[:10, 3] = 0.0  # ties in |u| handled like argmax (first index)
    u[10:20] = 1.0
    eta = torch.from_numpy(rng.integers(0, 3000, (5000, 3)).astype(np.int32)).cuda()
    want = ix.inv_perm.index_select(0, eta[:, 0].long()).long() * 256 + direction_bucket(u)
    assert torch.equal(ray_keys(u, eta, ix.inv_perm), want)
    want_mc = torch.arange(5000, device="cuda") // 7 * 256 + direction_bucket(u)
    assert torch.equal(ray_keys(u, rays_per_cell=7), want_mc)


def test_config2_full_size_properties():
    """BASELINE config 2 at full size (1e6 rays, N=20,000, d=6), through
    size-independent properties: (1) the pruned and exhaustive kernels agree
    bitwise on every ray (index, t, flag); (2) every hit point rp lies on the
    boundary between g and the hit generator with no generator strictly
    closer (nearest distance == |rp - x_g| == |rp - x_i| within the 1e-9
    coordinate tolerance -- the incircle property, checked against all N);
    (3) escaped rays have no generator in their forward halfspace."""
    import torch
    import bench
    pts = bench.generators()
    ns = vb.NodeSet(pts)
    s, p, u = bench.ray_recipe(10 ** 6)
    need = np.unique(p)
    sig_n, r_n = vb.descent_batch(ns, s[need], seed=0)
    pool_sig = np.zeros((bench.N_POOL, bench.DIM + 1), dtype=np.int32)
    pool_r = np.zeros((bench.N_POOL, bench.DIM))
    pool_sig[need], pool_r[need] = sig_n, r_n
    x, u, g = bench.assemble(pts, pool_sig, pool_r, p, u)
    xd, ud, gd = (torch.from_numpy(a).cuda() for a in (x, u, g))
    a = vb.raycast_batch(ns, xd, ud, gd, mode="pruned")
    b = vb.raycast_batch(ns, xd, ud, gd, mode="exhaustive")
    assert torch.equal(a.idx, b.idx) and torch.equal(a.flag, b.flag) and torch.equal(a.t, b.t)
    flag = a.flag.cpu().numpy()
    assert not (flag == 3).any() and not (flag == 2).any()
    ok = np.nonzero(flag == 0)[0]
    X = torch.from_numpy(pts).cuda()
    rp = a.rp[ok]
    rho = torch.linalg.norm(rp - X[gd[ok, 0].long()], dim=1)
    rho_i = torch.linalg.norm(rp - X[a.idx[ok].long()], dim=1)
    tol = 1e-9 * torch.clamp(rho, min=1.0)
    assert bool(((rho_i - rho).abs() <= tol).all())
    sample = ok[np.random.default_rng(0).choice(len(ok), 50000, replace=False)]
    _, d1, _ = ns._nearest_dev(a.rp[sample].cpu().numpy(), None)
    rs = torch.linalg.norm(a.rp[sample] - X[gd[sample, 0].long()], dim=1).cpu().numpy()
    assert np.all(np.abs(d1 - rs) <= 1e-9 * np.maximum(1.0, rs))
    esc = np.nonzero(flag == 1)[0]
    assert 0 < len(esc) < 2000
    ue = ud[esc]
    thr = (ue * X[gd[esc, 0].long()]).sum(1)
    thr = thr + 1e-12 * torch.clamp(thr.abs(), min=1.0)
    assert bool(((X @ ue.T).max(0).values <= thr).all())


@pytest.mark.parametrize("d", [4, 6, 8])
@pytest.mark.parametrize("case", ["offset", "anisotropic", "clustered"])
def test_fp32_screen_robust_to_scale(case, d):
    """The fp32 screen's and the tensor-core (tf32) screen's rigorous bounds
    must hold for badly scaled inputs: a large common offset
    (1e3 + 1e-3 * U), wildly different axis scales, and tight clusters.
    Pruned fp32 (FFMA2 at d = 4, tensor core at d = 6, 8) == exhaustive fp64
    bitwise."""
    rng = np.random.default_rng(77 + d)
    n = 6000
    if case == "offset":
        pts = 1e3 + 1e-3 * rng.random((n, d))
    elif case == "anisotropic":
        pts = rng.random((n, d)) * np.array([1e4, 1.0, 1e-4, 3e2, 10.0, 1e-2, 5.0, 0.1])[:d]
    else:
        centers = rng.random((20, d)) * 100
        pts = centers[rng.integers(0, 20, n)] + 1e-3 * rng.standard_normal((n, d))
    ns = vb.build_node_set(pts)
    m = 5000
    g = rng.integers(0, n, m)
    u = rng.standard_normal((m, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    a = vb.raycast_batch(ns, pts[g], u, g[:, None], mode="exhaustive", screen="fp64").to_host()
    for mode in ("pruned", "exhaustive"):
        b = vb.raycast_batch(ns, pts[g], u, g[:, None], mode=mode, screen="fp32").to_host()
        for x, y in zip(a, b):
            assert np.array_equal(x, y, equal_nan=True), mode
    want, _ = orc.raycast_argmin(pts, pts[g[:300]], u[:300], g[:300, None])
    got = a[0][:300]
    ok = a[3][:300] != 3
    assert np.array_equal(got[ok], want[ok])


def _tf32_rna(a):
    """cvt.rna.tf32.f32 restated in numpy: keep 10 explicit mantissa bits,
    round to nearest, ties away from zero."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x1000) & ~np.uint64(0x1FFF)).astype(np.uint32)
    return r.view(np.float32)


@pytest.mark.parametrize("d", [5, 6, 8])
def test_pack_records_mma_layout(d):
    """vr_pack_records_mma writes the rec32 features [x~, |x~|^2, 1, 0..]
    (sentinel |x~|^2 -> 1e30), tf32-rounded, in mma.sync m16n8k8 B-fragment
    order: [tile][block of 8][k-step][lane][2], lane l holding features
    8s + (l & 3) and 8s + (l & 3) + 4 of candidate 8 * block + (l >> 2)."""
    pts = np.random.default_rng(40 + d).standard_normal((1000, d))
    ns = vb.NodeSet(pts)
    ix = ns.prune_index()
    rec32 = ix.rec32rows.cpu().numpy()
    rows = rec32.shape[0]
    ks = (d + 2 + 7) // 8
    feat = np.zeros((rows, 8 * ks), dtype=np.float32)
    feat[:, :d] = rec32[:, :d]
    sq = rec32[:, d].copy()
    sq[np.isinf(sq)] = 1e30
    feat[:, d] = sq
    feat[:, d + 1] = 1.0
    feat = _tf32_rna(feat)
    lane = np.arange(32)
    want = np.empty((rows // 64, 8, ks, 32, 2), dtype=np.float32)
    for s in range(ks):
        for blk in range(8):
            cand = np.arange(rows // 64)[:, None] * 64 + 8 * blk + (lane >> 2)[None, :]
            want[:, blk, s, :, 0] = feat[cand, 8 * s + (lane & 3)]
            want[:, blk, s, :, 1] = feat[cand, 8 * s + (lane & 3) + 4]
    got = ix.recB.cpu().numpy().reshape(want.shape)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


_MMA_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2405_10050_b200 as vb
out = []
for n, d, seed in ((20000, 6, 0), (30000, 8, 1), (8000, 5, 2)):
    pts = np.random.default_rng(seed).random((n, d))
    ns = vb.NodeSet(pts)
    rng = np.random.default_rng(seed + 10)
    g = rng.integers(0, n, 20000).astype(np.int32)
    u = rng.standard_normal((20000, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    out += list(vb.raycast_batch(ns, pts[g], u, g[:, None], mode="pruned").to_host())
np.savez(sys.argv[2], *out)
"""


def test_tensor_core_screen_matches_ffma2_screen(tmp_path):
    """The tensor-core screen (default from d = 5) and the packed-FFMA2 fp32
    screen (VR_MMA=0, read once per process, hence subprocesses) return
    bitwise-identical results on generator-start rays, d = 5, 6, 8."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("1", "0"):
        path = str(tmp_path / f"mma{mode}.npz")
        env = dict(os.environ, VR_MMA=mode)
        p = subprocess.run([sys.executable, "-c", _MMA_SCRIPT, root, path], env=env,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        res[mode] = np.load(path)
    for k in res["1"].files:
        assert np.array_equal(res["1"][k], res["0"][k], equal_nan=True), k
