"""Summarise an ncu 'cuda,sass' source CSV per CUDA source line: instructions executed and
warp-stall samples, sorted.  Usage: python tools/ncu_lines.py src.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
lines = {}
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # source line summary row
        try:
            ln = int(r[0])
        except ValueError:
            continue
        def num(name):
            v = r[hdr.index(name)]
            return int(v) if v.isdigit() else 0
        samp = num("Warp Stall Sampling (All Samples)")
        inst = num("Instructions Executed")
        lines[ln] = (inst, samp, r[1][:90])
tot_i = sum(v[0] for v in lines.values()) or 1
tot_s = sum(v[1] for v in lines.values()) or 1
print(f"total warp-instr {tot_i:,}  samples {tot_s:,}")
for ln, (i, s, src) in sorted(lines.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{ln:5d} inst {100*i/tot_i:5.1f}%  stall {100*s/tot_s:5.1f}%  {src}")
