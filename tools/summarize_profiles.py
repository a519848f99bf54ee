"""Summarise a profiling pass (tools/gpu_profile_all.sh) into profiles/: launch tables per
config, ncu --set full key metrics of the dominant kernel per config, and
profiles/ncu_traffic.json (DRAM bytes per launch of the bench's roofline kernel)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof")
tag = sys.argv[2] if len(sys.argv) > 2 else "r01s2"
out = []
traffic = {}
for cfg in (2, 3, 4, 5):
    lc = os.path.join(src, f"launches_c{cfg}.csv")
    if os.path.exists(lc):
        t = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_table.py"), lc],
                           capture_output=True, text=True).stdout
        out.append(f"## config {cfg}: eager launch list of one bench step (ncu gpu__time_duration, clock-control none)\n\n```\n{t}```\n")
    raw = os.path.join(src, f"full_c{cfg}_raw.csv")
    if os.path.exists(raw):
        rows = list(csv.reader(io.StringIO(open(raw).read())))
        h, u, v = rows[0], rows[1], rows[2]
        def g(k):
            return (v[h.index(k)], u[h.index(k)]) if k in h else ("-", "")
        name = g("Kernel Name")[0]
        dur = float(g("gpu__time_duration.sum")[0].replace(",", ""))
        dur_us = dur * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(g("gpu__time_duration.sum")[1], 1.0)
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(g("dram__bytes_read.sum")[0].replace(",", "")) * mult.get(g("dram__bytes_read.sum")[1], 1)
        wr = float(g("dram__bytes_write.sum")[0].replace(",", "")) * mult.get(g("dram__bytes_write.sum")[1], 1)
        traffic[f"config{cfg}" + ("_kr" if "k_persist" in name else "")] = rd + wr
        stalls = sorted(((float(v[i].replace(",", "")), k[33:]) for i, k in enumerate(h)
                         if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("_not_issued")
                         and v[i] not in ("", "n/a")), reverse=True)
        tot = sum(s for s, _ in stalls) or 1
        lines = [f"kernel: {name}", f"duration: {dur_us:.1f} us", f"DRAM read {rd/1e6:.1f} MB, write {wr/1e6:.1f} MB "
                 f"-> {(rd+wr)/dur_us/1e3:.0f} GB/s"]
        for k in ["launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__cluster_dim_x",
                  "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                  "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum"]:
            val, un = g(k)
            lines.append(f"{k}: {val} {un}")
        lines.append("top stall reasons: " + ", ".join(f"{k} {100*s/tot:.0f}%" for s, k in stalls[:6]))
        out.append(f"## config {cfg}: ncu --set full of the dominant kernel (one launch)\n\n```\n" + "\n".join(lines) + "\n```\n")
path = os.path.join(ROOT, "profiles", f"{tag}_summary.md")
open(path, "w").write(f"# Profiles {tag} (B200, sm_100a)\n\nSource: tools/gpu_profile_all.sh; raw CSVs beside this file.\n\n" + "\n".join(out))
tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
json.dump(traffic, open(tp, "w"), indent=1)
print(open(path).read()[-3000:])
print(traffic)
