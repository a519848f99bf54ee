"""Run W warm-up steps and K profiled steps of the bench workload (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1710_01758_b200 import SbPcg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--slices", type=int, default=0)
a = ap.parse_args()
spec, per, first = bench.workload(a.config, 1, 0, a.slices)
prm = spec.params
ph, sens, mask, noise = bench.make_inputs(a.config, first, per)
dev = torch.device("cuda", 0)
ctx = SbPcg(torch.from_numpy(sens).to(torch.complex64).to(dev), torch.from_numpy(mask).to(dev),
            prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
y = bench.kspace_gpu(ctx, spec, ph, torch.from_numpy(mask).to(dev), noise, dev)
for i in range(a.warmup + a.steps):
    if i == a.warmup:
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    ctx.build_precond()
    x, log = ctx.recon(y, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters, precond=1,
                       use_graph=not a.eager)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("pcg iters per step", sum(sum(r) for r in log["pcg_iters"]), "launches", ctx.launches())
