"""Warp-level instructions (x32 per pixel) and stall samples by source-line range of edge.cu
(ncu cuda,sass CSV).  Usage: python tools/ncu_phase_warp.py src.csv npx name:a-b ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
px = float(sys.argv[2])
cur, hdr, agg, smp = None, None, {}, {}
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    v = r[hdr.index("Instructions Executed")]
    w = r[hdr.index("Warp Stall Sampling (All Samples)")]
    agg[(cur, int(r[0]))] = int(v) if v.isdigit() else 0
    smp[(cur, int(r[0]))] = int(w) if w.isdigit() else 0
T = sum(agg.values())
S = sum(smp.values()) or 1
print(f"total warp inst x32/px {32 * T / px:.1f}")
rest_i, rest_s = T, S
for spec in sys.argv[3:]:
    name, rng = spec.split(":")
    f = "edge.cu"
    if "@" in name:
        name, f = name.split("@")
    a, b = (int(x) for x in rng.split("-"))
    i = sum(v for (ff, l), v in agg.items() if ff == f and a <= l <= b)
    sm = sum(v for (ff, l), v in smp.items() if ff == f and a <= l <= b)
    rest_i -= i
    rest_s -= sm
    print(f"{name:14s} inst {32 * i / px:7.1f}/px  stall {100 * sm / S:5.1f}%")
print(f"{'rest':14s} inst {32 * rest_i / px:7.1f}/px  stall {100 * rest_s / S:5.1f}%")
