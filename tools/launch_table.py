"""Per-kernel mean duration from an ncu --metrics gpu__time_duration.sum --csv log.
Usage: python tools/launch_table.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h is None or len(r) < len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    agg.setdefault(d["Kernel Name"][:70], []).append(float(d["Metric Value"].replace(",", "")))
tot = sum(sum(v) for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:72s} n={len(v):5d} mean={sum(v) / len(v) / 1000:9.2f} us  share={100 * sum(v) / tot:5.1f}%")
