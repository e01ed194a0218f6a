"""Group an ncu 'cuda,sass' source CSV (edge kernel) by phase: per-file line ranges ->
instructions executed and stall samples.  Usage: python tools/ncu_groups.py src.csv"""
import csv
import sys

GROUPS = [  # (file suffix, first line, last line, name) -- edge.cu ranges as of round 2
    ("edge.cu", 294, 351, "gray"),
    ("edge.cu", 353, 427, "blur"),
    ("edge.cu", 429, 504, "sobel"),
    ("edge.cu", 517, 594, "nms_decide"),
    ("edge.cu", 596, 628, "nms_finish"),
    ("edge.cu", 630, 726, "band_loop"),
    ("edge.cu", 728, 1137, "median_collect_select"),
    ("edge.cu", 1138, 1217, "apply"),
    ("edge.cu", 1219, 1444, "scheduler"),
    ("edge.cu", 1, 293, "helpers"),
    ("igs_common.cuh", 1, 10000, "common(hypot,..)"),
]
cur = None
hdr = None
agg = {}
for r in csv.reader(open(sys.argv[1])):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
        hdr = None
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    ln = int(r[0])
    num = lambda k: int(r[hdr.index(k)]) if r[hdr.index(k)].isdigit() else 0
    inst = num("Instructions Executed")
    samp = num("Warp Stall Sampling (All Samples)")
    name = "other:" + cur.rsplit("/", 1)[-1]
    for suf, a, b, g in GROUPS:
        if cur.endswith(suf) and a <= ln <= b:
            name = g
            break
    i0, s0 = agg.get(name, (0, 0))
    agg[name] = (i0 + inst, s0 + samp)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr {ti:,}  stall samples {ts:,}")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:24s} inst {100 * i / ti:5.1f}%  ({i / 203.36e6:5.2f}/px)  samples {100 * s / ts:5.1f}%")
