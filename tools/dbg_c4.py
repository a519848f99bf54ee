"""Config-4: tolerance-mode SB recon per-slice iteration counts at FULL batch, plane path vs
generic path vs the oracle on sampled slices."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from oracle import problems, sb

NS = int(os.environ.get("NS", "256"))
SAMPLE = [0, 97, 200]
n_out = int(os.environ.get("NOUT", "6"))
if len(sys.argv) > 1:
    import bench
    from paper_1710_01758_b200 import SbPcg
    q = synth.problem_c4(range(NS))
    prm = synth.CONFIGS[4].params
    dev = torch.device("cuda", 0)
    ctx = SbPcg(torch.from_numpy(q["sens"]).cuda(), torch.from_numpy(q["mask"]).cuda(), prm.mu, prm.lam, prm.gamma, 3)
    ys = np.stack([problems.make_kspace(q["phantom"][i], q["sens"][i].astype(np.complex128), q["mask"],
                                        q["noise"][i].astype(np.complex128)) for i in SAMPLE])
    y = bench.kspace_gpu(ctx, synth.CONFIGS[4], q["phantom"], torch.from_numpy(q["mask"]).cuda(), q["noise"], dev)
    for k, i in enumerate(SAMPLE):  # the sampled slices use the oracle's k-space
        y[i] = torch.from_numpy(ys[k]).to(torch.complex64).cuda()
    x, log = ctx.recon(y, n_out, eps=1e-4, max_iters=50)
    it = np.array(log["pcg_iters"])
    np.save(f"gpurun_out/dbg_c4_{sys.argv[1]}.npy", x.cpu().numpy()[SAMPLE])
    print(sys.argv[1], "total", it.sum(), "sampled", json.dumps(it[:, SAMPLE].T.tolist()))
    sys.exit(0)
for mode, env in (("plane", {}), ("generic", {"SBPCG_NO_PLANE": "1"})):
    subprocess.run([sys.executable, __file__, mode], env={**os.environ, **env}, check=True)
q = synth.problem_c4(SAMPLE)
prm = synth.CONFIGS[4].params
for k, i in enumerate(SAMPLE):
    s32 = q["sens"][k].astype(np.complex128)
    y = problems.make_kspace(q["phantom"][k], s32, q["mask"], q["noise"][k].astype(np.complex128))
    x, log = sb.sb_recon(y.astype(np.complex64).astype(np.complex128), s32, q["mask"], prm.mu, prm.lam, prm.gamma,
                         n_out, 1, 3, 1e-4, 50, "circulant")
    print("oracle slice", i, log.pcg_iters)
    for mode in ("plane", "generic"):
        g = np.load(f"gpurun_out/dbg_c4_{mode}.npy")[k]
        print("  ", mode, "relerr vs oracle", np.linalg.norm(g - x) / np.linalg.norm(x))
