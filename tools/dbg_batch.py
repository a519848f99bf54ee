"""Tolerance-mode SB recon at a given batch for config CFG; sampled slices vs the oracle."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from oracle import problems, sb
from paper_1710_01758_b200 import SbPcg

CFG = int(os.environ.get("CFG", "3"))
NS = int(os.environ.get("NS", "128"))
n_out = int(os.environ.get("NOUT", "4"))
SAMPLE = [0, NS // 2, NS - 1]
spec = synth.CONFIGS[CFG]
prm = spec.params
if CFG == 4:
    q = synth.problem_c4(range(NS))
    sens, mask = q["sens"], q["mask"]
    ph = q["phantom"]; noise = q["noise"]
else:
    ps = [synth.problem2d(CFG, s) for s in range(NS)]
    sens = np.stack([p["sens"] for p in ps]).astype(np.complex64)
    mask = np.stack([p["mask"] for p in ps])
    ph = np.stack([p["phantom"] for p in ps]); noise = np.stack([p["noise"] for p in ps])
ctx = SbPcg(torch.from_numpy(sens).cuda(), torch.from_numpy(mask).cuda(), prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
ys = []
for i in range(NS):
    m = mask if mask.ndim == 2 else mask[i]
    ys.append(problems.make_kspace(ph[i], sens[i].astype(np.complex128), m, noise[i].astype(np.complex128)))
y = torch.from_numpy(np.stack(ys)).to(torch.complex64).cuda()
x, log = ctx.recon(y, n_out, eps=1e-4, max_iters=50)
it = np.array(log["pcg_iters"])
xs = x.cpu().numpy()
worst = 0.0
for i in SAMPLE:
    m = mask if mask.ndim == 2 else mask[i]
    s32 = sens[i].astype(np.complex128)
    xr, lg = sb.sb_recon(ys[i].astype(np.complex64).astype(np.complex128), s32, m, prm.mu, prm.lam, prm.gamma,
                         n_out, 1, prm.wavelet_levels, 1e-4, 50, "circulant")
    e = np.linalg.norm(xs[i] - xr) / np.linalg.norm(xr)
    worst = max(worst, e)
    print(f"cfg{CFG} NS={NS} G={os.environ.get('SBPCG_K1_G','auto')} plane={os.environ.get('SBPCG_NO_PLANE','0')} slice {i}: gpu {it[:, i].tolist()} oracle {lg.pcg_iters} relerr {e:.2e}")
print("WORST", worst)
