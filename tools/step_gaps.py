"""Where the config-2 bench step's device time goes between the library's own work: CUDA events
around build_precond and recon (host-enqueued, as bench.py times them) against the library's
internal Lambda-build and recon event times, plus the host time of each call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1710_01758_b200 import SbPcg  # noqa: E402

spec = synth.CONFIGS[2]
p = synth.problem2d(2, 0)
prm = spec.params
ctx = SbPcg(torch.from_numpy(p["sens"][None]).to(torch.complex64).cuda(), torch.from_numpy(p["mask"][None]).cuda(),
            prm.mu, prm.lam, prm.gamma, prm.wavelet_levels)
y = ctx.encode(torch.from_numpy(p["phantom"][None]).to(torch.complex64).cuda())
out = torch.empty_like(y[:, 0])
st = torch.cuda.current_stream()
rows = []
for rep in range(25):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record(st)
    h0 = time.perf_counter()
    ctx.build_precond()
    h1 = time.perf_counter()
    e[1].record(st)
    _, log = ctx.recon(y, prm.n_outer, eps=prm.eps, max_iters=prm.max_iters, out=out)
    h2 = time.perf_counter()
    e[2].record(st)
    e[2].synchronize()
    if rep >= 5:
        rows.append((e[0].elapsed_time(e[1]) * 1e3, e[1].elapsed_time(e[2]) * 1e3, log["build_s"] * 1e6,
                     log["total_ms"] * 1e3, (h1 - h0) * 1e6, (h2 - h1) * 1e6))
n = len(rows)
avg = [sum(r[i] for r in rows) / n for i in range(6)]
print("us: ev(build)=%.1f ev(recon)=%.1f lib build_s=%.1f lib recon total=%.1f host build call=%.1f host recon call=%.1f"
      % tuple(avg))
