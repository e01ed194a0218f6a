"""Thread instructions per pixel by source-line range of edge.cu (ncu cuda,sass CSV).
Usage: python tools/ncu_phases.py src.csv npx name:a-b [name:a-b ...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
px = float(sys.argv[2])
cur, hdr, agg = None, None, {}
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    v = r[hdr.index("Thread Instructions Executed")]
    agg[(cur, int(r[0]))] = int(v) if v.isdigit() else 0
print(f"total thread inst/px {sum(agg.values()) / px:.1f}")
for spec in sys.argv[3:]:
    name, rng = spec.split(":")
    f = "edge.cu"
    if "@" in name:
        name, f = name.split("@")
    a, b = (int(x) for x in rng.split("-"))
    print(f"{name:18s} {sum(v for (ff, l), v in agg.items() if ff == f and a <= l <= b) / px:7.1f}")
print("by file:", {f: round(sum(v for (ff, l), v in agg.items() if ff == f) / px, 1)
                   for f in sorted({k[0] for k in agg})})
