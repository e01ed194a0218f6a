"""Group an ncu 'cuda,sass' source CSV of the edge kernel by the enclosing function of each
edge.cu line (ranges found from the current source).  Usage: python tools/ncu_funcs.py src.csv [edge.cu]"""
import csv
import re
import sys

src = sys.argv[2] if len(sys.argv) > 2 else "paper_2603_08661_b200/csrc/edge.cu"
starts = []
for i, line in enumerate(open(src), 1):
    m = re.match(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__|static __device__)[^(]*?(\w+)\(", line)
    if m:
        starts.append((i, m.group(1)))
def func_of(ln):
    name = "file-scope"
    for a, n in starts:
        if a <= ln:
            name = n
        else:
            break
    return name
cur = hdr = None
agg = {}
for r in csv.reader(open(sys.argv[1])):
    if len(r) >= 2 and r[0] == "File Path":
        cur, hdr = r[1], None
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iI = hdr.index("Instructions Executed")
    s = int(r[iS]) if r[iS].isdigit() else 0
    e = int(r[iI]) if r[iI].isdigit() else 0
    key = func_of(int(r[0])) if cur.endswith("edge.cu") else "other:" + cur.rsplit("/", 1)[-1]
    a0, b0 = agg.get(key, (0, 0))
    agg[key] = (a0 + e, b0 + s)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr {ti:,} ({ti / 203.36e6:.2f}/px)  stall samples {ts:,}")
for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{k:28s} inst {i / 203.36e6:6.3f}/px  samples {s:7d} ({100 * s / ts:5.1f}%)")
