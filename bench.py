#!/usr/bin/env python
"""Headline benchmark: batched incircle RayCast, SURVEY.md §8(d) config 2.

Workload (BASELINE.json configs[1]): N=20,000 generators uniform in [0,1]^6
(default_rng(0)), 1,000,000 rays per GPU.  Ray k starts at the Voronoi vertex
reached by `descent` from generator s[p_k] (s = default_rng(1).choice(20000,
10000), p = default_rng(2).integers), with direction default_rng(3) normal
normalised, entering cell g = argmax_{s in sigma} u.x_s (eta = (g,)).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`ours`: one step = one fused RayCast launch (+ its exact re-check pass) over
the rank's 1e6 HBM-resident rays; value = all ranks' rays / max-over-ranks
device time.  `e2e` repeats the step through the public host-array API
(pinned host rays in, idx/t/rp/flag back out, copies inside the timed region).
`reference`: the reference's CPU algorithm (the oracle port of
raycast_incircle, kd-tree probe as in the reference for N > 2048) on all host
cores, on a bounded sample of the same rays per step.
"""

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # CPU legs: one BLAS thread per process

import argparse  # noqa: E402
import json  # noqa: E402
import multiprocessing as mp  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GEN, DIM, N_POOL, RAYS_PER_GPU = 20000, 6, 10000, 1_000_000
METRIC = "RayCast rays/sec (config 2: d=6, N=20000)"
FLOP_PER_PAIR = 2 * DIM  # incircle-sphere screen: d FMAs per (ray, generator)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--rays", type=int, default=RAYS_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rays-per-core", type=int, default=3000)
    ap.add_argument("--mode", choices=["pruned", "exhaustive"], default="pruned")
    ap.add_argument("--no-extra", action="store_true", help="skip configs 1, 3, 4, 5")
    return ap.parse_args()


def generators():
    return np.random.default_rng(0).random((N_GEN, DIM))


def ray_recipe(n_total):
    """Start pool indices, pool pick per ray, unit directions (first 1e6 rays
    are exactly config 2; further ranks extend the same streams)."""
    s = np.random.default_rng(1).choice(N_GEN, N_POOL, replace=False)
    p = np.random.default_rng(2).integers(0, N_POOL, n_total)
    u = np.random.default_rng(3).standard_normal((n_total, DIM))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    return s, p, u


def assemble(pts, pool_sig, pool_r, p, u):
    x = pool_r[p]
    sig = pool_sig[p]
    proj = np.einsum("kd,ksd->ks", u, pts[sig])
    g = sig[np.arange(len(p)), np.argmax(proj, axis=1)].astype(np.int32)
    return np.ascontiguousarray(x), np.ascontiguousarray(u), np.ascontiguousarray(g[:, None])


# --------------------------------------------------------------------------
# CPU legs (oracle port of the reference algorithm; test infrastructure)
# --------------------------------------------------------------------------
_W = {}


def _w_init(pts):
    from oracle import voronray_oracle as orc
    _W["orc"] = orc
    _W["nodes"] = orc.Nodes(pts)


def _w_descent(start):
    orc = _W["orc"]
    sig, r = orc.descent(_W["nodes"], int(start), orc.stream(0, "descent", int(start)))
    return sig, r


def _w_rays(args):
    x, u, g = args
    orc = _W["orc"]
    out = np.full(len(g), -1, dtype=np.int64)
    for k in range(len(g)):
        res = orc.raycast(_W["nodes"], (int(g[k]),), x[k], u[k])
        if res is not None:
            out[k] = [s for s in res[0] if s != int(g[k])][0]
    return out


def cpu_pool(pts, cores):
    ctx = mp.get_context("fork")
    return ctx.Pool(cores, initializer=_w_init, initargs=(pts,))


def cpu_rays(pool, x, u, g, cores):
    chunks = max(1, cores * 4)
    bounds = np.linspace(0, len(g), chunks + 1).astype(int)
    jobs = [(x[a:b], u[a:b], g[a:b, 0]) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    t0 = time.perf_counter()
    parts = pool.map(_w_rays, jobs)
    return np.concatenate(parts), time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md clocks line)
# --------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.3)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
def fma_peak(torch, L, _lib, dtype=0):
    """DFMA (dtype 0) / FFMA (dtype 1) pipe peak, or the tf32 mma.sync peak
    (dtype 2), measured live (MEASURED_PEAKS.json has no FP64 / FP32 / tf32
    figure)."""
    scratch = torch.empty(16, dtype=torch.float64, device="cuda")
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sm * 8, (4096 if dtype < 2 else 512)
    per = 4096.0 if dtype < 2 else 131072.0
    best = 0.0
    sh = _lib.stream_handle()
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.vr_fma_probe(dtype, blocks, iters, _lib.ptr(scratch), sh))
        e1.record()
        e1.synchronize()
        best = max(best, per * iters * blocks / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def _median_passes(fn, passes, torch, reset=None):
    """Run fn() `passes` times (device-synchronised wall time each); the
    first pass pays one-off costs (lazy module loading, allocator growth) and
    is listed but excluded; the median of the rest is reported."""
    times, out = [], None
    for rep in range(passes + 1):
        if reset is not None and rep:
            reset()
        out = None  # the previous pass's result is freed first: its device
        # blocks are what this pass's allocations reuse (otherwise two passes'
        # tables coexist and the first timed passes pay for cudaMalloc)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    return float(np.median(times[1:])), times, out


def _w_edge_rays(args):
    """Oracle raycasts of traversal edge rays: hit index per ray (-1 escape)."""
    x, u, eta = args
    orc = _W["orc"]
    out = np.full(len(x), -1, dtype=np.int64)
    for k in range(len(x)):
        e = tuple(int(v) for v in eta[k])
        res = orc.raycast(_W["nodes"], e, x[k], u[k])
        if res is not None:
            out[k] = [s for s in res[0] if s not in e][0]
    return out


def _w_mc_cells(args):
    cells, z, n = args
    orc = _W["orc"]
    vols = []
    for c, zc in zip(cells, z):
        try:
            _, v, _ = orc.mc_areas(_W["nodes"], int(c), n, orc.Replay(zc))
        except orc.Escaped:
            v = float("nan")
        vols.append(v)
    return np.array(vols)


def cpu_pool_shared(nodes, cores):
    """Pool whose workers inherit an already-built oracle node set (fork)."""
    from oracle import voronray_oracle as orc
    _W["orc"], _W["nodes"] = orc, nodes
    return mp.get_context("fork").Pool(cores)


def cpu_edge_rays(pts, mesh, vb, torch, n_rays, cores, seed):
    """The reference's CPU RayCast (oracle port, kd-tree probe loop for N >
    2048) on a random sample of the traversal's own edge rays, on all host
    cores; returns (rays/s, sample size, index agreement with the GPU)."""
    from oracle import voronray_oracle as orc
    dv = mesh.device_arrays()
    V, d = dv["r"].shape
    rng = np.random.default_rng(seed)
    nv = max(1, n_rays // (d + 1))
    pick = torch.as_tensor(np.sort(rng.choice(V, nv, replace=False)), device=dv["r"].device)
    sig = dv["sigma"][pick].contiguous()
    r = dv["r"][pick].cpu().numpy()
    ns = mesh.nodes
    u, ok = vb.vertex_directions_batch(ns, sig)
    u, ok, sig = u.cpu().numpy(), ok.cpu().numpy().astype(bool), sig.cpu().numpy()
    xs, us, etas = [], [], []
    for k in range(d + 1):
        keep = ok[:, k]
        xs.append(r[keep])
        us.append(u[keep, k])
        etas.append(np.delete(sig[keep], k, axis=1))
    x, uu, eta = np.concatenate(xs), np.concatenate(us), np.concatenate(etas)
    gpu = vb.raycast_batch(ns, x, uu, eta.astype(np.int32), want_rp=False)
    gidx = gpu.idx.cpu().numpy()
    nodes = orc.Nodes(pts)
    pool = cpu_pool_shared(nodes, cores)
    try:
        bounds = np.linspace(0, len(x), cores * 4 + 1).astype(int)
        jobs = [(x[a:b], uu[a:b], eta[a:b]) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        t0 = time.perf_counter()
        got = np.concatenate(pool.map(_w_edge_rays, jobs))
        wall = time.perf_counter() - t0
    finally:
        pool.close()
        pool.join()
    return len(x) / wall, len(x), float(np.mean(got == gidx))


def extra_configs(vb, torch, world, rank, cpu=True, passes=5):
    """The other SURVEY §8(d) configs, measured in the same run: each is run
    `passes` + 1 times (device-synchronised wall time; the first pass is
    excluded) and the median reported.  Configs 3 and 5 are also timed from
    the raw point array (NodeSet construction + the native kd index build +
    the traversal), like the reference whose cKDTree is built inside
    NodeSet.__init__.  With `cpu`, the reference's CPU path (the oracle port)
    is timed on this box's host cores in the same run: config 1 as-is (one
    core: the reference DFS is sequential), configs 3 and 5 on a sample of
    their own edge rays, config 4 on a sample of cells (replayed Philox
    normals).  Multi-rank: the traversal levels are ray-sharded, MC cells are
    sharded."""
    from paper_2405_10050_b200 import parallel
    from oracle import voronray_oracle as orc
    import hashlib
    cores = host_cores()
    out = {}

    def digest(sig):
        return hashlib.sha256(np.ascontiguousarray(sig[np.lexsort(sig.T[::-1])], dtype="<i4")
                              .tobytes()).hexdigest()

    # ---- config 1: full diagram N=1000, d=3 ------------------------------
    pts1 = np.random.default_rng(0).random((1000, 3))
    ns1 = vb.build_node_set(pts1)
    # a few ms of mostly host-side latency: 12x the passes, so that a burst of
    # host scheduling noise (one run had its first 13 passes at 4-60 ms, the
    # rest at 3.1 ms) does not set the median
    p1 = 12 * passes
    med, ts, (m1, info1) = _median_passes(
        lambda: vb.voronoi_graph(ns1, seed=0, return_info=True), p1, torch)
    c1 = {"vertices": info1["vertices"], "seconds": med, "passes_s": ts,
          "timing": f"median of {p1} passes after one warm pass",
          "vertices_per_s": info1["vertices"] / med, "levels": len(info1["levels"]),
          "sigma_digest_matches_reference": digest(m1.arrays()["sigma"]) ==
          "b1f6f8721369b9116ff154e6673225998fb3785479bb65c18dafb6b2db2c0b1a"}
    if cpu:
        t0 = time.perf_counter()
        verts, _, _, _ = orc.voronoi_graph(orc.Nodes(pts1), seed=0)
        wall = time.perf_counter() - t0
        c1["cpu_baseline"] = {"seconds": wall, "cores": 1, "kind": "port",
                              "sample": "the whole config (oracle DFS voronoi_graph, one core: "
                                        "the reference traversal is sequential)",
                              "vertices": len(verts), "speedup": wall / med}
    out["config1_full_diagram"] = c1

    # ---- config 3: full diagram N=10,000, d=5 ----------------------------
    pts3 = np.random.default_rng(0).standard_normal((10000, 5))
    ns3 = vb.build_node_set(pts3)
    ns3.prune_index()
    w3 = torch.zeros(16, dtype=torch.int64, device="cuda")
    med, ts, (m3, info3) = _median_passes(
        lambda: vb.voronoi_graph(ns3, seed=0, return_info=True, work=w3), passes, torch,
        reset=lambda: w3.zero_())

    def from_points3():
        ns = vb.build_node_set(pts3)
        t0 = time.perf_counter()
        ns.prune_index()
        torch.cuda.synchronize()
        bt = time.perf_counter() - t0
        m = vb.voronoi_graph(ns, seed=0)
        return m, bt
    med_fp, ts_fp, (_, bt3) = _median_passes(from_points3, passes, torch)
    t0 = time.perf_counter()
    sig = m3.arrays()["sigma"]  # host materialisation of the device-resident mesh
    dt_host = time.perf_counter() - t0
    c3 = {"vertices": info3["vertices"], "seconds": med, "passes_s": ts,
          "timing": f"median of {passes} passes after one warm pass",
          "vertices_per_s": info3["vertices"] / med,
          "seconds_from_points": med_fp, "passes_from_points_s": ts_fp,
          "index_build_s": bt3,
          "mesh": "device-resident (HBM); host arrays + sorted edges materialised on first access",
          "host_materialise_s": dt_host,
          "sigma_digest_matches_reference": digest(sig) ==
          "f8093583cb129297758ebea66c8fcbbf3938086d9f8b8ee1b0f79096a9351173",
          "pairs_screened": int(w3[0].item()), "d": 5}
    if cpu:
        rate, m, agree = cpu_edge_rays(pts3, m3, vb, torch, 400 * cores, cores, 3)
        st3 = vb.RaycastStats()
        vb.voronoi_graph(ns3, seed=0, stats=st3)
        c3["cpu_baseline"] = {"rays_per_s": rate, "cores": cores, "kind": "port",
                              "sample": f"{m} edge rays of the config-3 mesh (random vertices, "
                                        "all their edges), oracle raycast_incircle (kd-tree probe)",
                              "index_agreement": agree,
                              "projected_seconds": st3.raycasts / rate,
                              "projection": "the traversal's edge raycasts at this rate (the "
                                            "reference DFS is one core: x cores)"}
    out["config3_full_diagram"] = c3
    del m3

    # ---- config 4: MC, 1e5 cells x 1000 rays, d=4 -----------------------
    pts4 = np.random.default_rng(0).random((100000, 4))
    ns4 = vb.NodeSet(pts4)
    ns4.prune_index()
    cells = np.arange(100000)
    w4 = torch.zeros(16, dtype=torch.int64, device="cuda")
    med, ts, res4 = _median_passes(
        lambda: parallel.mc_cells_sharded(ns4, cells, 1000, seed=0, work=w4), passes, torch,
        reset=lambda: w4.zero_())
    c4 = {"cells": 100000, "rays_per_cell": 1000, "seconds": med, "passes_s": ts,
          "timing": f"median of {passes} passes after one warm pass",
          "rays_per_s": 1e8 / med, "bounded_cells": int((res4.status == 0).sum()),
          "pairs_screened": int(w4[0].item()), "d": 4}
    if cpu:
        sub = np.random.default_rng(4).choice(100000, 6 * cores, replace=False)
        z = vb.mc_directions(4, sub, 1000, seed=0).reshape(len(sub), 1000, 4)
        pool = cpu_pool_shared(orc.Nodes(pts4), cores)
        try:
            bounds = np.linspace(0, len(sub), cores + 1).astype(int)
            jobs = [(sub[a:b], z[a:b], 1000) for a, b in zip(bounds[:-1], bounds[1:])]
            t0 = time.perf_counter()
            vols = np.concatenate(pool.map(_w_mc_cells, jobs))
            wall = time.perf_counter() - t0
        finally:
            pool.close()
            pool.join()
        gv = res4.volume[sub]
        okc = np.isfinite(vols) & (res4.status[sub] == 0)
        rel = np.abs(vols[okc] - gv[okc]) / np.abs(gv[okc])
        c4["cpu_baseline"] = {"rays_per_s": len(sub) * 1000 / wall, "cores": cores,
                              "kind": "port",
                              "sample": f"{len(sub)} random cells x 1000 rays, oracle mc_areas "
                                        "(per-ray raycast path) on the device's Philox normals",
                              "max_rel_volume_diff_vs_gpu": float(rel.max()) if rel.size else None,
                              "projected_seconds": 1e8 / (len(sub) * 1000 / wall)}
    out["config4_mc"] = c4
    del res4, ns4  # config 5 needs ~60 GB of level tables
    torch.cuda.empty_cache()

    # ---- config 5: L=5 local traversal of 10,000 seeds, N=1e6, d=8 ------
    pts5 = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
    ns5 = vb.NodeSet(pts5)
    ns5.prune_index()
    seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
    w5 = torch.zeros(16, dtype=torch.int64, device="cuda")
    st5 = vb.RaycastStats()
    keep = {}

    def run5():
        # the previous pass's mesh is released first; its ~50 GB of level
        # tables come back from torch's caching allocator (steady state, as
        # in a serving process), so the passes measure the traversal and not
        # cudaMalloc of fresh tables
        keep.clear()
        keep["m"], keep["lv"] = vb.voronoi_local(ns5, seeds, hops=5, stats=st5,
                                                 return_levels=True, work=w5)

    def reset5():
        w5.zero_()
        st5.raycasts = st5.nn_calls = st5.iterations = 0
    med, ts, _ = _median_passes(run5, passes, torch, reset=reset5)
    m5, lv = keep["m"], keep["lv"]

    def from_points5():
        keep.clear()
        t0 = time.perf_counter()
        ns = vb.NodeSet(pts5)
        ns.prune_index()
        torch.cuda.synchronize()
        keep["bt"] = time.perf_counter() - t0
        keep["m"] = vb.voronoi_local(ns, seeds, hops=5)
    med_fp, ts_fp, _ = _median_passes(from_points5, 3, torch)
    bt5 = keep["bt"]
    keep.clear()
    torch.cuda.empty_cache()
    m5 = vb.voronoi_local(ns5, seeds, hops=5)
    # parity at bench scale: the reference L=5 balls of the first 20 seeds
    # (tests/golden/config5_balls_l5.npz) are contained in this vertex set,
    # and verify_vertex holds on a random 10k sample
    balls_ok, verify_ok = None, None
    gpath = os.path.join(ROOT, "tests", "golden", "config5_balls_l5.npz")
    if os.path.exists(gpath):
        gz = np.load(gpath)
        balls_ok = bool(all(m5.contains(gz[f"ball{m}_sigma"]).all() for m in range(20)))
    dv = m5.device_arrays()
    pick = torch.as_tensor(np.sort(np.random.default_rng(7).choice(dv["sigma"].shape[0], 10000,
                                                                   replace=False)),
                           device=dv["sigma"].device)
    verify_ok = bool(vb.verify_vertices(ns5, dv["sigma"][pick].cpu().numpy(),
                                        dv["r"][pick].cpu().numpy()).all())
    c5 = {"seeds": 10000, "hops": 5, "vertices": int(len(lv)), "seconds_incl_descent": med,
          "passes_s": ts, "timing": f"median of {passes} passes after one warm pass",
          "seconds_from_points": med_fp, "passes_from_points_s": ts_fp,
          "index_build_s": bt5,
          "mesh": "device-resident (HBM), not copied to the host",
          "pairs_screened": int(w5[0].item()), "d": 8,
          "vertices_per_s": len(lv) / med,
          "edge_raycasts_this_rank": st5.raycasts,
          "per_level": np.bincount(lv).tolist(),
          "checks": {"config5_balls_ok": balls_ok, "config5_verify_ok": verify_ok,
                     "balls": "20 reference L=5 balls (tests/golden/config5_balls_l5.npz) "
                              "contained in the vertex set",
                     "verify": "verify_vertices on 10,000 random vertices"}}
    if cpu:
        rate, m, agree = cpu_edge_rays(pts5, m5, vb, torch, 150 * cores, cores, 5)
        c5["cpu_baseline"] = {"rays_per_s": rate, "cores": cores, "kind": "port",
                              "sample": f"{m} edge rays of the config-5 vertex set (random "
                                        "vertices, all their edges), oracle raycast_incircle "
                                        "(kd-tree probe)", "index_agreement": agree,
                              "projected_seconds": c5["edge_raycasts_this_rank"] / rate}
    out["config5_local_traversal"] = c5
    return out


def profiled_traffic():
    """dram read + write bytes per launch of the dominant kernel, from the
    committed ncu --set full capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "r2_k_raycast_pruned_ncu_full.txt")
    if not os.path.exists(path):
        return None
    tot = 0.0
    for line in open(path):
        for key, scale in (("dram read", 1e6), ("dram write", 1e6)):
            if line.strip().startswith(key):
                parts = line.split()
                val, unit = float(parts[2]), parts[3]
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                tot += val * mult
    return tot or None


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2405_10050_b200 as vb
    from paper_2405_10050_b200 import _lib
    from paper_2405_10050_b200.raycast import HostRaycaster, Workspace

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # VR_DIST_BACKEND=gloo is a functional check of the multi-rank path on a
    # box with fewer GPUs than ranks (ranks share a GPU; no kernel waits on
    # another rank, the collectives run on the host) -- its numbers mean nothing
    backend = os.environ.get("VR_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    L = _lib.lib()

    pts = generators()
    ns = vb.build_node_set(pts)
    n = args.rays
    s, p_all, u_all = ray_recipe(n * world)
    lo, hi = rank * n, (rank + 1) * n
    # vertex pool: the reference descent (same host RNG streams), run on the GPU
    need = np.unique(p_all[lo:hi])
    t0 = time.perf_counter()
    sig_n, r_n = vb.descent_batch(ns, s[need], seed=0)
    t_pool = time.perf_counter() - t0
    pool_sig = np.zeros((N_POOL, DIM + 1), dtype=np.int32)
    pool_r = np.zeros((N_POOL, DIM))
    pool_sig[need], pool_r[need] = sig_n, r_n
    x, u, g = assemble(pts, pool_sig, pool_r, p_all[lo:hi], u_all[lo:hi])

    dev = torch.device("cuda", local)
    xd, ud, gd = (torch.from_numpy(a).to(dev) for a in (x, u, g))
    out = dict(idx=torch.empty(n, dtype=torch.int32, device=dev),
               t=torch.empty(n, dtype=torch.float64, device=dev),
               rp=torch.empty((n, DIM), dtype=torch.float64, device=dev),
               flag=torch.empty(n, dtype=torch.uint8, device=dev))
    ws = Workspace()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
          for _ in range(args.warmup + args.steps)]
    work = torch.zeros(16, dtype=torch.int64, device=dev)  # VR_WORK_COUNTERS
    ns.prune_index()  # kd index built once per NodeSet, outside the timing

    def step(i, mode=args.mode, events=None):
        flush.fill_(i & 0xFF)  # L2 flush, outside the timed events
        torch.cuda.nvtx.range_push("bench_step")  # ncu --nvtx-include "bench_step/"
        vb.raycast_batch(ns, xd, ud, gd, out=out, workspace=ws, events=events or ev[i],
                         mode=mode, work=work if mode == "pruned" else None)
        torch.cuda.nvtx.range_pop()

    for i in range(args.warmup):
        step(i)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.warmup, args.warmup + args.steps):
            step(i)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [ev[i][0].elapsed_time(ev[i][2]) for i in range(args.warmup, args.warmup + args.steps)]
    kern_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in range(args.warmup, args.warmup + args.steps)]
    screened = int(work[0].item()) / (args.warmup + args.steps) if args.mode == "pruned" else None
    wk = (work.double().cpu() / (args.warmup + args.steps)).tolist()
    n_warps = (n + 31) // 32
    counters = {"tiles_per_warp": wk[0] / (64 * 32) / n_warps,
                "tree_node_tests_per_warp": wk[5] / n_warps,
                "rare_blocks_per_warp": wk[1] / n_warps,
                "rare_iters_per_warp": wk[2] / n_warps,
                "rare_entries_per_ray": wk[3] / n, "sphere_updates_per_ray": wk[4] / n}
    if any(wk[6:11]):  # VR_RARE_STATS builds: rare-path entry outcomes per ray
        counters["rare_outcomes_per_ray"] = dict(zip(
            ("outside", "self", "behind", "band", "improves"), [v / n for v in wk[6:11]]))
    # the exhaustive (TMA-staged, unpruned) kernel on the same rays, for its
    # roofline: fp64 screen (FP64 pipe) and fp32 screen (FP32 pipe)
    ex_ms = {}
    for scr in ("fp64", "fp32"):
        ex_ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        flush.fill_(7)
        vb.raycast_batch(ns, xd, ud, gd, out=out, workspace=ws, mode="exhaustive", screen=scr)
        flush.fill_(8)
        vb.raycast_batch(ns, xd, ud, gd, out=out, workspace=ws, mode="exhaustive", screen=scr,
                         events=ex_ev)
        torch.cuda.synchronize()
        ex_ms[scr] = ex_ev[0].elapsed_time(ex_ev[1])
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    value = world * n * args.steps / (total_ms * 1e-3)

    # correctness guard on the timed outputs (cheap, outside the timing)
    flags = out["flag"].cpu().numpy()
    n_deg = int((flags == 3).sum())
    n_esc = int((flags == 1).sum())

    # ---- e2e through the public host-array API ----------------------------
    hr = HostRaycaster(ns, n, 1)
    hx, hu, hg = (HostRaycaster.pinned(a.shape, t) for a, t in
                  ((x, torch.float64), (u, torch.float64), (g, torch.int32)))
    hx.copy_(torch.from_numpy(x))
    hu.copy_(torch.from_numpy(u))
    hg.copy_(torch.from_numpy(g))
    hidx = HostRaycaster.pinned((n,), torch.int32)
    ht = HostRaycaster.pinned((n,), torch.float64)
    hrp = HostRaycaster.pinned((n, DIM), torch.float64)
    hfl = HostRaycaster.pinned((n,), torch.uint8)
    for _ in range(max(1, args.warmup)):
        hr.run(hx, hu, hg, hidx, ht, hrp, hfl, mode=args.mode)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hr.run(hx, hu, hg, hidx, ht, hrp, hfl, mode=args.mode)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world * n * args.steps / (float(e2e_t.item()) * 1e-3)
    assert np.array_equal(hidx.numpy(), out["idx"].cpu().numpy()), "e2e result differs"
    h2d = x.nbytes + u.nbytes + g.nbytes
    d2h = n * (4 + 8 + 8 * DIM + 1)

    extra = None
    if not args.no_extra:
        extra = extra_configs(vb, torch, world, rank, cpu=(world == 1 and not args.no_cpu_baseline))

    result = None
    if rank == 0:
        peak64 = fma_peak(torch, L, _lib, 0)
        peak32 = fma_peak(torch, L, _lib, 1)
        mma_on = os.environ.get("VR_MMA", "1") != "0"
        peak_tc = fma_peak(torch, L, _lib, 2) if mma_on else None
        kms = float(np.mean(kern_ms))
        pairs = screened if screened is not None else n * N_GEN
        achieved = pairs * FLOP_PER_PAIR / (kms * 1e-3) / 1e12
        ex64 = n * N_GEN * FLOP_PER_PAIR / (ex_ms["fp64"] * 1e-3) / 1e12
        ex32 = n * N_GEN * FLOP_PER_PAIR / (ex_ms["fp32"] * 1e-3) / 1e12
        traffic = profiled_traffic()
        tc_on = mma_on and args.mode == "pruned"
        # FFMA-equivalent view: the screen's d-dot (2d flop per screened
        # pair) against the live FFMA peak (the packed-FFMA2 build's pipe)
        cuda_core = {"bound": "fp32", "achieved": achieved, "peak": peak32, "unit": "TFLOP/s",
                     "frac": achieved / peak32, "flop_per_pair": FLOP_PER_PAIR,
                     "peak_source": "measured live: FFMA probe (vr_fma_probe dtype 1)"}
        common = {"traffic": traffic,
                  "kernel": ("k_raycast_pruned<6,R=1,tile=64,tensor-core screen>" if tc_on else
                             "k_raycast_pruned<6,R=1,tile=64,fp32 screen>"
                             if args.mode == "pruned" else "k_raycast<6,2,128,256,4,3>"),
                  "kernel_ms": kms, "pairs_per_launch": pairs, "pairs_per_ray": pairs / n,
                  "work_counters": counters if args.mode == "pruned" else None,
                  "screen": ("tensor-core (mma.sync tf32: sphere + halfspace products) + fp64 rare path"
                             if tc_on else "packed FFMA2 fp32 + fp64 rare path"),
                  "unit_of_work": "(ray, generator) pair screened; the pruned kernel counts "
                                  "the pairs it actually screened (work counter)",
                  "traffic_source": "profiles/r2_k_raycast_pruned_ncu_full.txt",
                  "note": "latency-bound (tree walk, fp64 rare path): neither pipe saturates; "
                          "see DESIGN.md section 2"}
        if tc_on:
            # the screen runs on the warp tensor path: its tf32 product
            # [z, 1, c] . [x, |x|^2, 1] is 2 (d + 2) flop per screened pair
            tc_ach = pairs * 2 * (DIM + 2) / (kms * 1e-3) / 1e12
            roofline = {"bound": "tensor", "achieved": tc_ach, "peak": peak_tc, "unit": "TFLOP/s",
                        "frac": tc_ach / peak_tc, "flop_per_pair": 2 * (DIM + 2),
                        "peak_source": "measured live: tf32 mma.sync m16n8k8 probe (vr_fma_probe "
                                       "dtype 2), the instruction the screen issues",
                        "frac_of_tcgen05_tf32_nominal": tc_ach / 1100.0,
                        "cuda_core_equivalent": cuda_core, **common}
        else:
            roofline = {**cuda_core, **common}
        result = {
            "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config-2 recipe, SURVEY.md §8(d))",
            "config": arm_config(world, n),
            "roofline": roofline,
            "roofline_exhaustive": {
                "fp64_screen": {"bound": "fp64", "kernel_ms": ex_ms["fp64"], "achieved": ex64,
                                "peak": peak64, "unit": "TFLOP/s", "frac": ex64 / peak64,
                                "rays_per_s": n / (ex_ms["fp64"] * 1e-3)},
                "fp32_screen": {"bound": "fp32", "kernel_ms": ex_ms["fp32"], "achieved": ex32,
                                "peak": peak32, "unit": "TFLOP/s", "frac": ex32 / peak32,
                                "rays_per_s": n / (ex_ms["fp32"] * 1e-3)},
                "kernel": "k_raycast<6,2,128,256,4,3> (TMA ring, every pair screened)",
                "pairs_per_launch": n * N_GEN},
            "e2e": {"value": e2e_value, "unit": "rays/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "HostRaycaster.run (pinned host arrays)"},
            "gpu_launches": (3 if args.mode == "pruned" else 2) * args.steps,  # [ray keys +] RayCast + re-check
            "clocks": clk.summary(),
            "checks": {"escaped": n_esc, "degenerate": n_deg, "pool_build_s": t_pool},
        }
        if extra is not None:
            for key, ent in extra.items():
                if "pairs_screened" in ent:
                    secs = ent.get("seconds", ent.get("seconds_incl_descent"))
                    fl = 2 * ent["d"]
                    ach = ent["pairs_screened"] * fl / secs / 1e12
                    ent["roofline"] = {
                        "bound": "fp32", "flop_per_pair": fl, "achieved": ach, "peak": peak32,
                        "unit": "TFLOP/s", "frac": ach / peak32,
                        "time_basis": "whole-config wall time (all phases), so a lower "
                                      "bound on the pruned kernel's own rate"}
            result["extra_configs"] = extra
        if world == 1 and not args.no_cpu_baseline:
            cores = host_cores()
            m = min(n, args.cpu_rays_per_core * cores)
            pool = cpu_pool(pts, cores)
            try:
                cpu_idx, wall = cpu_rays(pool, x[:m], u[:m], g[:m], cores)
            finally:
                pool.close()
                pool.join()
            agree = float(np.mean(cpu_idx == out["idx"].cpu().numpy()[:m]))
            result["cpu_baseline"] = {
                "value": m / wall, "unit": "rays/s", "cores": cores, "kind": "port",
                "sample": f"first {m} config-2 rays, oracle raycast (kd-tree probe loop), "
                          f"{cores} processes", "index_agreement": agree}
    if world > 1:
        dist.destroy_process_group()
    return result


def arm_config(world, n):
    """The `config` object of both arms (same workload, same keys)."""
    return {"workload": "config2: batched RayCast N=20000 d=6, 1e6 rays/GPU from "
                        "descent vertices, eta=(g,)",
            "n_generators": N_GEN, "d": DIM, "rays_per_gpu": n,
            "parallelism": f"ray-sharded x{world}, generators replicated",
            "l2": "flushed between timed steps (256 MB write, untimed)"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    cores = host_cores()
    pts = generators()
    m = min(args.rays, args.cpu_rays_per_core * cores)
    s, p_all, u_all = ray_recipe(m * (args.warmup + args.steps))
    pool = cpu_pool(pts, cores)
    try:
        need = np.unique(p_all)
        res = pool.map(_w_descent, s[need], chunksize=max(1, len(need) // (cores * 4)))
        pool_sig = np.zeros((N_POOL, DIM + 1), dtype=np.int32)
        pool_r = np.zeros((N_POOL, DIM))
        for k, (sg, r) in zip(need, res):
            pool_sig[k], pool_r[k] = sg, r
        times = []
        for i in range(args.warmup + args.steps):
            sl = slice(i * m, (i + 1) * m)
            x, u, g = assemble(pts, pool_sig, pool_r, p_all[sl], u_all[sl])
            _, wall = cpu_rays(pool, x, u, g, cores)
            if i >= args.warmup:
                times.append(wall)
    finally:
        pool.close()
        pool.join()
    value = m * args.steps / sum(times)
    return {"metric": METRIC, "value": value, "unit": "rays/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded config-2 recipe, SURVEY.md §8(d))",
            "config": arm_config(world, args.rays),
            "cpu_baseline": {"value": value, "unit": "rays/s", "cores": cores, "kind": "port",
                             "sample": f"{m} config-2 rays per step (the first rays of the same "
                                       "recipe), oracle restatement of raycast_incircle "
                                       "(kd-tree probe loop, scipy cKDTree)"},
            "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
