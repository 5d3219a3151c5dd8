"""Workload for the per-kernel ncu table (tools/kernel_table.py): one pass of
each config's device path -- config 2 (1e6 descent-vertex rays, N=20k, d=6),
config 4 (MC, 1e5 cells x 1000 rays, d=4), config 1 (full diagram, N=1000,
d=3: the persistent small-level kernel), config 3 (full diagram, N=1e4,
d=5), config 5 (L=5 balls around 10k seeds, N=1e6, d=8).  Run under ncu
with -k regex:^k_ (our kernels only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_10050_b200 as vb  # noqa: E402

torch.cuda.set_device(0)
pts = bench.generators()
ns = vb.build_node_set(pts)
n = 1_000_000
s, p_all, u_all = bench.ray_recipe(n)
need = np.unique(p_all)
sig_n, r_n = vb.descent_batch(ns, s[need], seed=0)
pool_sig = np.zeros((bench.N_POOL, bench.DIM + 1), dtype=np.int32)
pool_r = np.zeros((bench.N_POOL, bench.DIM))
pool_sig[need], pool_r[need] = sig_n, r_n
x, u, g = bench.assemble(pts, pool_sig, pool_r, p_all, u_all)
xd, ud, gd = (torch.from_numpy(a).cuda() for a in (x, u, g))
ns.prune_index()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("config2")
vb.raycast_batch(ns, xd, ud, gd)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()

pts4 = np.random.default_rng(0).random((100000, 4))
ns4 = vb.NodeSet(pts4)
ns4.prune_index()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("config4")
res = vb.mc_cells(ns4, np.arange(100000), 1000, seed=0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()

pts1 = np.random.default_rng(0).random((1000, 3))
ns1 = vb.build_node_set(pts1)
vb.voronoi_graph(ns1, seed=0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("config1")
vb.voronoi_graph(ns1, seed=0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()

pts3 = np.random.default_rng(0).standard_normal((10000, 5))
ns3 = vb.build_node_set(pts3)
ns3.prune_index()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("config3")
vb.voronoi_graph(ns3, seed=0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()

pts5 = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns5 = vb.NodeSet(pts5)
ns5.prune_index()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("config5")
mesh, lv = vb.voronoi_local(ns5, seeds, hops=5, return_levels=True)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok", len(lv))
