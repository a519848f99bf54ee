"""bench.py's own run with the binding's update_sens / recon wrapped by host timers: where the
e2e leg's step time goes (host time per call, the library's device recon time)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import bench  # noqa: E402
from paper_1710_01758_b200 import SbPcg  # noqa: E402

acc = {"us": [], "rc": [], "dev": [], "host": []}
_us, _rc = SbPcg.update_sens, SbPcg.recon


def us(self, s):
    t = time.perf_counter()
    r = _us(self, s)
    if not s.is_cuda:
        acc["us"].append(time.perf_counter() - t)
    return r


def rc(self, y, *a, **k):
    t = time.perf_counter()
    r = _rc(self, y, *a, **k)
    if not y.is_cuda:
        acc["rc"].append(time.perf_counter() - t)
        acc["dev"].append(r[1]["total_ms"])
    return r


SbPcg.update_sens, SbPcg.recon = us, rc
sys.argv = ["bench.py", "--steps", "20", "--warmup", "5", "--no-extra", "--no-cpu-baseline"]
bench.main()
import statistics as st  # noqa: E402
for k, v in acc.items():
    if v:
        v = v[3:]
        sc = 1.0 if k == "dev" else 1e3
        print(k, "n", len(v), "median %.3f mean %.3f max %.3f ms" % (sc * st.median(v), sc * st.mean(v), sc * max(v)), file=sys.stderr)
