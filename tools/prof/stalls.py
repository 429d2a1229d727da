"""Summarise an ncu source-page CSV (--page source --csv --print-source sass): stall reasons and
the hottest SASS instructions. usage: python tools/prof/stalls.py src.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in cols}
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot, seen, hot = Counter(), set(), []
for r in rows[2:]:
    if len(r) < len(hdr) or r[ia] in seen:
        continue
    seen.add(r[ia])
    for h in cols:
        try:
            tot[h] += int(r[idx[h]] or 0)
        except ValueError:
            pass
    try:
        hot.append((int(r[iss] or 0), r[ia], r[isrc].strip()))
    except ValueError:
        pass
s = sum(tot.values()) or 1
print("stall reasons (% of samples):")
for h, v in tot.most_common():
    if v:
        print(f"  {h:28s} {100 * v / s:5.1f}%")
print("hottest instructions:")
S = sum(h[0] for h in hot) or 1
for v, a, src in sorted(hot, reverse=True)[:top]:
    print(f"  {100 * v / S:5.1f}%  {a[-5:]}  {src[:90]}")
