"""Summarise tools/gpu_pipes.sh: per config, the dominant kernel's mean over the profiled launches
of duration, DRAM bytes, FMA-pipe busy %, issue-active %, warps-active % -> profiles/ncu_pipes.json;
DRAM bytes per launch -> profiles/ncu_traffic.json (key configN, or configN_kr for k_persist)."""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "pipes")
tag = sys.argv[2] if len(sys.argv) > 2 else "r02"
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
        "ms": 1e3, "msecond": 1e3, "%": 1.0, "inst": 1.0, "": 1.0}
out, traffic = {}, json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
for cfg in (2, 3, 4, 5):
    path = os.path.join(src, f"c{cfg}.csv")
    if not os.path.exists(path):
        continue
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    per = defaultdict(dict)
    name = None
    for r in rows[1:]:
        v = float(r[ix["Metric Value"]].replace(",", "")) * mult.get(r[ix["Metric Unit"]], 1.0)
        per[r[ix["ID"]]][r[ix["Metric Name"]]] = v
        name = r[ix["Kernel Name"]]
    keys = set().union(*[set(d) for d in per.values()])
    mean = {k: sum(d.get(k, 0.0) for d in per.values()) / len(per) for k in keys}
    dram = mean["dram__bytes_read.sum"] + mean["dram__bytes_write.sum"]
    out[f"config{cfg}"] = {
        "kernel": name, "launches": len(per), "duration_us": mean["gpu__time_duration.sum"],
        "dram_bytes": dram, "dram_gbs": dram / mean["gpu__time_duration.sum"] / 1e3,
        "fma_pipe_busy_pct": mean["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"],
        "issue_active_pct": mean["smsp__issue_active.avg.pct_of_peak_sustained_active"],
        "warps_active_pct": mean["sm__warps_active.avg.pct_of_peak_sustained_active"],
        "fma_inst_share": mean["sm__inst_executed_pipe_fma.sum"] / max(mean["smsp__inst_executed.sum"], 1.0),
        "source": f"ncu --metrics (tools/gpu_pipes.sh), {tag}, mean of {len(per)} launches, clock-control none"}
    traffic[f"config{cfg}_kr" if "k_persist" in name else f"config{cfg}"] = dram
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_pipes.json"), "w"), indent=1)
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
