"""Config-2 A/B of the pruned-path kernels (env VR_SWEEP / VR_MMA select):
median kernel time over 5 L2-flushed steps, work counters, and bitwise
agreement with the exhaustive fp64 kernel on the same rays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_10050_b200 as vb  # noqa: E402
from paper_2405_10050_b200.raycast import Workspace  # noqa: E402


def main(n=int(os.environ.get("NRAYS", "1000000"))):
    dev = torch.device("cuda", 0)
    pts = bench.generators()
    ns = vb.build_node_set(pts)
    s, p_all, u_all = bench.ray_recipe(n)
    need = np.unique(p_all)
    sig_n, r_n = vb.descent_batch(ns, s[need], seed=0)
    pool_sig = np.zeros((bench.N_POOL, bench.DIM + 1), dtype=np.int32)
    pool_r = np.zeros((bench.N_POOL, bench.DIM))
    pool_sig[need], pool_r[need] = sig_n, r_n
    x, u, g = bench.assemble(pts, pool_sig, pool_r, p_all, u_all)
    xd, ud, gd = (torch.from_numpy(a).to(dev) for a in (x, u, g))
    ws = Workspace()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ns.prune_index()
    ts, ks = [], []
    for i in range(8):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        work = torch.zeros(16, dtype=torch.int64, device=dev)
        flush.fill_(i)
        torch.cuda.nvtx.range_push("ab")
        res = vb.raycast_batch(ns, xd, ud, gd, workspace=ws, events=ev, mode="pruned", work=work)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(ev[0].elapsed_time(ev[2]))
            ks.append(ev[0].elapsed_time(ev[1]))
    wk = work.double().cpu().numpy()
    ex = vb.raycast_batch(ns, xd, ud, gd, mode="exhaustive", screen="fp64")
    same = all(torch.equal(getattr(res, f), getattr(ex, f)) for f in ("idx", "flag")) and \
        torch.equal(torch.nan_to_num(res.t, posinf=1e300), torch.nan_to_num(ex.t, posinf=1e300))
    tag = f"VR_SWEEP={os.environ.get('VR_SWEEP', '-')} VR_HSWEEP={os.environ.get('VR_HSWEEP', '-')}"
    print(f"{tag}: step {np.median(ts):.3f} ms kernel {np.median(ks):.3f} ms  "
          f"pairs/ray {wk[0] / n:.0f} rare blocks/ray {wk[1] / n:.2f} entries/ray {wk[3] / n:.2f} "
          f"updates/ray {wk[4] / n:.2f} degenerate {int((res.flag == 3).sum())} "
          f"rare warp-steps/warp {wk[2] / (n / 32):.1f} equal_to_exhaustive={same}", flush=True)
    if any(wk[6:11]):
        print("  rare outcomes per ray:", dict(zip(("outside", "self", "behind", "band", "improves"),
                                                   np.round(wk[6:11] / n, 3))), flush=True)


if __name__ == "__main__":
    main()
