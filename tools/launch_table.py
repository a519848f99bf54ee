"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    k = r[4].split("(")[0].replace("void ", "") + " grid" + r[8]
    agg[k][0] += 1
    agg[k][1] += float(r[14]) / 1e3
tot = sum(v[1] for v in agg.values())
print(f"{'total us':>10} {'share':>6} {'n':>5} {'avg us':>8}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1]:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:5d} {v[1] / v[0]:8.2f}  {k}")
print(f"{tot:10.1f} total us over {len(rows)} launches")
