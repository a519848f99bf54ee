"""The paper's preconditioner comparison (Fig. 5a/5b analogue; SURVEY 8(f)
NEXT-1) on the GPU: config-2 geometry (256x256, 12 coils, VD lines R=4), parameter sets 1-3
(PAPER.md:270-274), eps = 1e-3 and 20 x 1 SB iterations, phantom x1e3 so the
shrinkage is active (readings A8, SURVEY 8(c) "several-fold" pin).  Reports total and
first-solve PCG iterations and the GPU recon time per preconditioner, and the oracle's
iteration counts for set 1 (none / circulant) beside them.  Output: gpurun_out/paper_sets.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import problems, sb  # noqa: E402
from paper_1710_01758_b200 import SbPcg  # noqa: E402

p = synth.problem2d(2, 0, amplitude=1e3)
y = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
names = {0: "none", 2: "jacobi", 1: "circulant"}
res = {}
for sid, (mu, lam, gam) in synth.PAPER_SET.items():
    ctx = SbPcg(torch.from_numpy(p["sens"][None]).to(torch.complex64).cuda(),
                torch.from_numpy(p["mask"][None]).cuda(), mu, lam, gam, 3)
    yt = torch.from_numpy(y[None]).to(torch.complex64).cuda()
    for pk in (0, 2, 1):
        ctx.recon(yt, 20, eps=1e-3, max_iters=200, precond=pk)  # warm-up (graph capture)
        torch.cuda.synchronize()
        t = time.perf_counter()
        x, log = ctx.recon(yt, 20, eps=1e-3, max_iters=200, precond=pk)
        dt = time.perf_counter() - t
        it = [r[0] for r in log["pcg_iters"]]
        res[f"set{sid}_{names[pk]}"] = dict(total=sum(it), first=it[0], per_outer=it, recon_ms=1e3 * dt)
    ctx.close()
    r = res
    print(f"set {sid} (mu,lam,gam)=({mu},{lam},{gam}): total none/jacobi/circulant = "
          f"{r[f'set{sid}_none']['total']}/{r[f'set{sid}_jacobi']['total']}/{r[f'set{sid}_circulant']['total']}"
          f"  ratio none/circ {r[f'set{sid}_none']['total'] / max(1, r[f'set{sid}_circulant']['total']):.2f}"
          f"  first solve {r[f'set{sid}_none']['first']}/{r[f'set{sid}_jacobi']['first']}/{r[f'set{sid}_circulant']['first']}"
          f"  recon ms {r[f'set{sid}_none']['recon_ms']:.1f}/{r[f'set{sid}_jacobi']['recon_ms']:.1f}/{r[f'set{sid}_circulant']['recon_ms']:.1f}")
if "--oracle" in sys.argv:
    mu, lam, gam = synth.PAPER_SET[1]
    for pk in ("none", "circulant"):
        _, lg = sb.sb_recon(y, p["sens"], p["mask"], mu, lam, gam, 20, 1, 3, 1e-3, 200, pk)
        res[f"oracle_set1_{pk}"] = dict(total=sum(lg.pcg_iters), first=lg.pcg_iters[0], per_outer=lg.pcg_iters)
        print("oracle set 1", pk, sum(lg.pcg_iters), lg.pcg_iters)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/paper_sets.json", "w"), indent=1)
