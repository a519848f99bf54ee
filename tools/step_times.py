"""Per-step SB recon device times (CUDA events) for a config, to see the distribution."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
from paper_1710_01758_b200 import SbPcg
cfg = int(os.environ.get("CFG", "2")); n = int(os.environ.get("N", "20"))
spec, per, first = bench.workload(cfg, 1, 0, 0)
prm = spec.params
ph, sens, mask, noise = bench.make_inputs(cfg, first, per)
dev = torch.device("cuda", 0)
mask_d = torch.from_numpy(mask).to(dev)
ctx = SbPcg(torch.from_numpy(sens).to(torch.complex64).to(dev), mask_d, prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
y = bench.kspace_gpu(ctx, spec, ph, mask_d, noise, dev)
flush = torch.empty(2 * bench.L2_BYTES // 4, dtype=torch.float32, device=dev)
ts = []
for i in range(n):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x, log = ctx.recon(y, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(os.environ.get("TAG", ""), "cfg", cfg, "ms per step:", " ".join(f"{t:.2f}" for t in ts), "| log total_ms", round(log["total_ms"], 2))
