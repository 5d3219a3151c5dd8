"""GPU-busy fraction of a traversal (union of kernel intervals from a CUPTI
trace vs the wall time of the call) and the idle gaps between kernels, for
config 3 (full diagram, N=1e4, d=5) and config 1.  Tells host / launch
latency apart from device time."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2405_10050_b200 as vb  # noqa: E402


def busy(fn, name):
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    path = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = sorted((e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
                if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e)
    union, cur_s, cur_e = 0.0, None, None
    gaps = []
    for s, e, _ in ks:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                union += cur_e - cur_s
                gaps.append(s - cur_e)
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        union += cur_e - cur_s
    span = (ks[-1][1] - ks[0][0]) if ks else 0.0
    gaps = np.array(gaps) if gaps else np.zeros(1)
    print(f"{name}: wall {wall * 1e3:.2f} ms, first->last kernel {span / 1e3:.2f} ms, "
          f"GPU busy {union / 1e3:.2f} ms ({len(ks)} kernels/copies), idle gaps: "
          f"{len(gaps)} totalling {gaps.sum() / 1e3:.2f} ms (>20us: {(gaps > 20).sum()}, "
          f"{gaps[gaps > 20].sum() / 1e3:.2f} ms)", flush=True)


def main():
    p3 = np.random.default_rng(0).standard_normal((10000, 5))
    ns3 = vb.build_node_set(p3)
    ns3.prune_index()
    busy(lambda: vb.voronoi_graph(ns3, seed=0), "config3 voronoi_graph")
    p1 = np.random.default_rng(0).random((1000, 3))
    ns1 = vb.build_node_set(p1)
    ns1.prune_index()
    busy(lambda: vb.voronoi_graph(ns1, seed=0), "config1 voronoi_graph")


if __name__ == "__main__":
    main()
