"""Stall reasons summed over an edge.cu line range of an ncu 'cuda,sass' source CSV.
Usage: python tools/ncu_stalls.py src.csv FIRST LAST"""
import csv
import sys
lo, hi = int(sys.argv[2]), int(sys.argv[3])
cur = hdr = None
agg = {}
for r in csv.reader(open(sys.argv[1])):
    if len(r) >= 2 and r[0] == "File Path":
        cur, hdr = r[1], None
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit() or not cur.endswith("edge.cu"):
        continue
    if not lo <= int(r[0]) <= hi:
        continue
    for k, v in zip(hdr, r):
        if k.startswith("stall_") and "Not Issued" not in k and v.isdigit():
            agg[k] = agg.get(k, 0) + int(v)
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"{k:24s} {v:7d} {100 * v / tot:5.1f}%")
