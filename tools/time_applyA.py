"""Time repeated apply_A (the matvec kernel alone) for a config, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1710_01758_b200 import SbPcg
cfg = int(os.environ.get("CFG", "4")); n = int(os.environ.get("N", "10"))
spec, per, first = bench.workload(cfg, 1, 0, 0)
prm = spec.params
ph, sens, mask, noise = bench.make_inputs(cfg, first, per)
dev = torch.device("cuda", 0)
ctx = SbPcg(torch.from_numpy(sens).to(torch.complex64).to(dev), torch.from_numpy(mask).to(dev), prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
x = torch.from_numpy(ph).to(torch.complex64).to(dev)
y = ctx.apply_A(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    ctx.apply_A(x, out=y)
e1.record(); e1.synchronize()
print(os.environ.get("TAG", ""), f"cfg{cfg} apply_A {e0.elapsed_time(e1) / n * 1e3:.1f} us")
