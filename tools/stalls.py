"""Stall breakdown of one ncu capture: per-reason cycles/issue from the raw page and the top
SASS instructions per reason from the source page (--print-source sass).
usage: python tools/stalls.py <raw.csv> <sass.csv> [n]"""
import csv
import sys

raw = list(csv.reader(open(sys.argv[1])))
d = dict(zip(raw[0], raw[2] if len(raw) > 2 else raw[1]))
pre = "smsp__average_warps_issue_stalled_"
st = {k[len(pre):].replace("_per_issue_active.ratio", ""): float(v) for k, v in d.items()
      if k.startswith(pre) and k.endswith("_per_issue_active.ratio")}
print("cycles per issued instruction by reason (total %.2f):" % sum(st.values()))
print("  " + ", ".join("%s %.2f" % kv for kv in sorted(st.items(), key=lambda x: -x[1]) if kv[1] >= 0.05))
for k in ["gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "dram__bytes_read.sum", "dram__bytes_write.sum"]:
    if k in d:
        print("  %s = %s" % (k, d[k]))
rows = list(csv.reader(open(sys.argv[2])))
h, data = rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
n = int(sys.argv[3]) if len(sys.argv) > 3 else 6


def f(r, k):
    try:
        return float(r[ix[k]])
    except (KeyError, ValueError):
        return 0.0


tot = {k: sum(f(r, k) for r in data) for k in h if k.startswith("stall_") and "Not" not in k}
for key, _ in sorted(tot.items(), key=lambda x: -x[1])[:6]:
    print("== %s (%d samples)" % (key, tot[key]))
    for r in sorted(data, key=lambda r: -f(r, key))[:n]:
        print("  %6d %s" % (f(r, key), r[ix["Source"]][:100]))
