"""Parse `ncu -i <rep> --page raw --csv` output: per-launch DRAM bytes and duration of the
captured kernel(s); writes/updates profiles/ncu_traffic.json {"config<N>": bytes per launch}."""
import csv
import io
import json
import os
import sys

rep_csv, cfg = sys.argv[1], sys.argv[2]
rows = list(csv.reader(io.StringIO(open(rep_csv).read())))
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "Kernel Name"]
out = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        rd = float(r[idx["dram__bytes_read.sum"]].replace(",", ""))
        wr = float(r[idx["dram__bytes_write.sum"]].replace(",", ""))
        du = float(r[idx["gpu__time_duration.sum"]].replace(",", ""))
    except (KeyError, ValueError):
        continue
    out.append(dict(kernel=r[idx["Kernel Name"]][:60], read=rd, write=wr, dur=du))
units = rows[1]
print("units:", units[idx["dram__bytes_read.sum"]], units[idx["gpu__time_duration.sum"]])
for o in out:
    print(o)
if out:
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[idx["dram__bytes_read.sum"]], 1)
    tot = sum(o["read"] + o["write"] for o in out) / len(out) * mult
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[f"config{cfg}"] = tot
    json.dump(d, open(path, "w"), indent=1)
    print("traffic per launch", tot)
