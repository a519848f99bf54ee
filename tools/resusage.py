"""Per-kernel registers / stack / shared memory of libsbpcg.so (cuobjdump -res-usage).
usage: python tools/resusage.py [regex]"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-res-usage", "paper_1710_01758_b200/libsbpcg.so"], capture_output=True,
                     text=True).stdout.splitlines()
pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
fn = None
for line in out:
    m = re.search(r"Function (\S+):", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
    if m and fn:
        dem = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        if pat.search(dem):
            print(f"{dem:60s} REG={m.group(1):>4} STACK={m.group(2):>4} SHARED={m.group(3):>5}")
        fn = None
