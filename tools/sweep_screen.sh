python - <<'PY' 2>&1 | grep -v Warn
import sys; sys.path.insert(0,".")
import numpy as np, torch, paper_2405_10050_b200 as vb
from tools.sweep_pruned import run
pts=np.random.default_rng(0).random((20000,6)); ns=vb.NodeSet(pts)
rng=np.random.default_rng(3); n=1000000
g=rng.integers(0,20000,n).astype(np.int32); u=rng.standard_normal((n,6)); u/=np.linalg.norm(u,axis=1,keepdims=True)
dev=torch.device("cuda",0)
xd,ud,gd=(torch.from_numpy(a).to(dev) for a in (pts[g],u,g[:,None].copy()))
ns.prune_index(); ns.screen32()
for mode in ["exhaustive","pruned"]:
  for screen in ["fp64","fp32"]:
    vb.raycast_batch(ns,xd,ud,gd,mode=mode,screen=screen)
    e=[torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize(); vb.raycast_batch(ns,xd,ud,gd,mode=mode,screen=screen,events=e); torch.cuda.synchronize()
    print(mode, screen, "kernel ms", e[0].elapsed_time(e[1]))
PY
