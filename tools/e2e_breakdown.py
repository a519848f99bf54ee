"""Config-2 e2e step (bench.py's e2e leg) split into its two public calls, each bracketed by a
device synchronise: update_sens (6.3 MB pinned H2D + transposition + Lambda build) and recon
(6.3 MB pinned H2D of the k-space, the reconstruction, 0.5 MB D2H), plus a bare pinned H2D copy
of the same bytes for the box's PCIe rate."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1710_01758_b200 import SbPcg  # noqa: E402

spec = synth.CONFIGS[2]
p = synth.problem2d(2, 0)
prm = spec.params
sens_h = torch.from_numpy(p["sens"][None]).to(torch.complex64).pin_memory()
mask_h = torch.from_numpy(p["mask"][None]).pin_memory()
ctx = SbPcg(sens_h, mask_h, prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
y_h = ctx.encode(torch.from_numpy(p["phantom"][None]).to(torch.complex64).cuda()).cpu().pin_memory()
x_h = torch.empty((1,) + tuple(spec.shape), dtype=torch.complex64).pin_memory()
dst = torch.empty_like(sens_h, device="cuda")
if os.environ.get("E2E_SECOND_CTX"):
    ctx0 = SbPcg(sens_h.cuda(), mask_h.cuda(), prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
    ctx0.recon(y_h.cuda(), prm.n_outer, eps=prm.eps, max_iters=prm.max_iters)
if os.environ.get("E2E_FLUSH"):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
t_us, t_rc, t_cp, t_all = [], [], [], []
for rep in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.update_sens(sens_h)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, lg = ctx.recon(y_h, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters, out=x_h)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dst.copy_(sens_h, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    ctx.update_sens(sens_h)
    ctx.recon(y_h, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters, out=x_h)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if rep >= 5:
        t_us.append(t1 - t0), t_rc.append(t2 - t1), t_cp.append(t3 - t2), t_all.append(t4 - t3)
med = lambda v: 1e3 * statistics.median(v)  # noqa: E731
nb = sens_h.numel() * 8
print(f"PCG iterations {sum(sum(r) for r in lg['pcg_iters'])}, library recon total_ms {lg['total_ms']:.3f}; update_sens (host maps) {med(t_us):.3f} ms; recon (host k-space, host image) {med(t_rc):.3f} ms; "
      f"both back to back {med(t_all):.3f} ms; bare pinned H2D of {nb} B {med(t_cp):.3f} ms "
      f"= {nb / statistics.median(t_cp) / 1e9:.1f} GB/s; back-to-back mean {1e3 * statistics.mean(t_all):.3f} ms, "
      f"max {1e3 * max(t_all):.3f} ms")
