"""Print SASS context (with stall samples) around given addresses of an ncu source CSV.
usage: python tools/prof/ctx.py src.csv addr_suffix [before] [after]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
seen, lst = set(), []
for r in rows[2:]:
    if len(r) >= len(hdr) and r[ia] not in seen:
        seen.add(r[ia])
        lst.append(r)
b = int(sys.argv[3]) if len(sys.argv) > 3 else 12
a = int(sys.argv[4]) if len(sys.argv) > 4 else 4
for k, r in enumerate(lst):
    if r[ia].endswith(sys.argv[2]):
        for rr in lst[max(0, k - b):k + a]:
            print(rr[ia][-5:], rr[iss].rjust(6), rr[isrc][:110])
