"""The paper's preconditioner comparison (Fig. 5a/5b analogue; SURVEY 8(f)
NEXT-1) on the GPU: config-2 geometry (256x256, 12 coils, VD lines R=4), parameter sets 1-3
(PAPER.md:270-274), eps = 1e-3 and 20 x 1 SB iterations, phantom x1e3 so the
shrinkage is active (readings A8, SURVEY 8(c) "several-fold" pin).  Reports total and
first-solve PCG iterations and the GPU recon time per preconditioner (none / Jacobi /
circulant).

Two coil-map models:
  * "normalised": Sigma_c |S_c|^2 = 1 everywhere (BASELINE's model) -- diag(A) is then constant and
    Jacobi is a pure rescaling (identical iteration counts to no preconditioner);
  * "support": the paper's model: S_hat = S / sqrt(Sigma |S|^2) inside the
    subject's support and 0 outside (sb_normalize_sens), with a posterior-array-like coil set
    (the ring's coils on one half only), so diag(A) = mu f Sigma|S_hat|^2 + 4 lambda + gamma
    takes two values and Jacobi is a non-trivial diagonal scaling.
k-space is formed with the library's encoder (sb_encode) plus noise, as in bench.py.  The
oracle's counts for the same comparison are pinned by tests/test_gpu_paper_sets.py.
Output: gpurun_out/paper_sets.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1710_01758_b200 import SbPcg, normalize_sens  # noqa: E402


def support_of(phantom, grow=3):
    """Pixels of the subject (|phantom| > 0) dilated by `grow` pixels (periodic)."""
    s = np.abs(phantom) > 0
    out = s.copy()
    for dy in range(-grow, grow + 1):
        for dx in range(-grow, grow + 1):
            out |= np.roll(np.roll(s, dy, 0), dx, 1)
    return out.astype(np.uint8)


def kspace(ctx, x, mask, noise):
    yf = ctx.encode(torch.from_numpy(x[None]).to(torch.complex64).cuda(), full=True)
    sigma = 0.005 * yf.abs().amax()
    yf.add_(sigma * torch.from_numpy(noise[None]).to(torch.complex64).cuda())
    return yf * torch.from_numpy(mask[None, None]).to(torch.complex64).cuda()


def run(model):
    p = synth.problem2d(2, 0, amplitude=1e3)
    sens = torch.from_numpy(p["sens"][None]).to(torch.complex64).cuda()
    mask = p["mask"]
    if model == "support":
        C = sens.shape[1]
        keep = list(range(C // 2))  # posterior-array-like: half of the ring
        sens = sens[:, keep].contiguous()
        sup = torch.from_numpy(support_of(p["phantom"])).cuda()
        sens = normalize_sens(sens, sup)
    names = {0: "none", 2: "jacobi", 1: "circulant"}
    res = {}
    for sid, (mu, lam, gam) in synth.PAPER_SET.items():
        ctx = SbPcg(sens, torch.from_numpy(mask[None]).cuda(), mu, lam, gam, 3, persistent=False)
        yt = kspace(ctx, p["phantom"], mask, p["noise"][: sens.shape[1]])
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
        print(f"[{model}] set {sid} (mu,lam,gam)=({mu},{lam},{gam}): total none/jacobi/circulant = "
              f"{r[f'set{sid}_none']['total']}/{r[f'set{sid}_jacobi']['total']}/{r[f'set{sid}_circulant']['total']}"
              f"  ratio none/circ {r[f'set{sid}_none']['total'] / max(1, r[f'set{sid}_circulant']['total']):.2f}"
              f"  first solve {r[f'set{sid}_none']['first']}/{r[f'set{sid}_jacobi']['first']}/"
              f"{r[f'set{sid}_circulant']['first']}  recon ms {r[f'set{sid}_none']['recon_ms']:.1f}/"
              f"{r[f'set{sid}_jacobi']['recon_ms']:.1f}/{r[f'set{sid}_circulant']['recon_ms']:.1f}", flush=True)
    return res


if __name__ == "__main__":
    out = {m: run(m) for m in ("normalised", "support")}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/paper_sets.json", "w"), indent=1)
