"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum]
--csv): time share per kernel, and when the DRAM metrics were collected, DRAM bytes per launch and the
achieved DRAM rate (serialised, cold-cache launches: compare shares, not absolutes).
usage: python tools/prof/launches.py launches.csv [skip_first_n]"""
import csv
import re
import sys
from collections import defaultdict

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iname, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
iu = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
launch = defaultdict(dict)
names = {}
for r in rows[1:]:
    lid = int(r[iid])
    if lid < skip:
        continue
    v = float(r[iv].replace(",", "")) * (UNIT.get(r[iu], 1.0) if iu is not None else 1.0)
    launch[lid][r[iname]] = v
    names[lid] = re.sub(r"\(.*", "", r[ik])
tot, cnt, dram = defaultdict(float), defaultdict(int), defaultdict(float)
for lid, m in launch.items():
    k = names[lid]
    tot[k] += m.get("gpu__time_duration.sum", 0.0)
    cnt[k] += 1
    dram[k] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
T = sum(tot.values())
has_dram = any(dram.values())
print(f"total {T / 1e6:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    line = f"{100 * v / T:6.2f}%  {v / 1e3:10.1f} us  n={cnt[k]:6d}  avg={v / cnt[k] / 1e3:8.2f} us"
    if has_dram:
        b = dram[k] / cnt[k]
        line += f"  dram/launch={b / 1e6:9.3f} MB  {b / (v / cnt[k]):8.1f} GB/s"
    print(f"{line}  {k[:80]}")
