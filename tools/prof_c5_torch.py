import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2405_10050_b200 as vb
pts = np.random.default_rng(0).random((10 ** 6, 8)).astype(np.float32).astype(np.float64)
ns = vb.NodeSet(pts); ns.prune_index(); ns.screen32()
seeds = np.random.default_rng(1).choice(10 ** 6, 10000, replace=False)
vb.voronoi_local(ns, seeds[:100], hops=2)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=False) as prof:
    vb.voronoi_local(ns, seeds, hops=4)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
