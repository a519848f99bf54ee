"""Segment profile of the persistent kernel's PCG loop (SBPCG_KR_PROF=1): config-2 recon,
ns per iteration of each loop segment as seen by CTA 0 of problem 0."""
import os
import sys

os.environ.setdefault("SBPCG_KR_PROF", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1710_01758_b200 import SbPcg  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = synth.CONFIGS[cfg]
p = synth.problem2d(cfg, 0)
prm = spec.params
ctx = SbPcg(torch.from_numpy(p["sens"][None]).to(torch.complex64).cuda(), torch.from_numpy(p["mask"][None]).cuda(),
            prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
x = torch.from_numpy(p["phantom"][None]).to(torch.complex64).cuda()
y = ctx.encode(x)
for rep in range(3):
    xo, log = ctx.recon(y, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters)
    torch.cuda.synchronize()
    its = sum(sum(r) for r in log["pcg_iters"])
    print(f"rep {rep}: {log['total_ms']:.3f} ms, {its} PCG iterations, stages {log['stages']}", flush=True)
