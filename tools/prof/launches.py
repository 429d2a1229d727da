"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time share per kernel.
usage: python tools/prof/launches.py launches.csv [skip_first_n]"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iname = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1 + skip:]:
    if r[iname] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ik])
    name = re.sub(r"<(\d+), 1, 1, 16, 3, (\d)>", r"<MT\1,mode\2>", name)
    v = float(r[iv].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T/1e6:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{100*v/T:6.2f}%  {v/1e3:10.1f} us  n={cnt[k]:6d}  avg={v/cnt[k]/1e3:8.2f} us  {k[:90]}")
