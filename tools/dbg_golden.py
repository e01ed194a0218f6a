"""Debug: run the golden edge cases through the library in IGS_LIB, print mismatch details."""
import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from conftest import load_golden
import paper_2603_08661_b200 as b
E = load_golden("edge")
for case in sorted(E)[:6]:
    c = E[case]
    img = c["image"]
    if min(img.shape[:2]) < 3: continue
    got = b.importance_pipeline(img, float(c["sigma"]))
    want = c["importance"]
    bad = np.argwhere(~((got == want) | (np.isnan(got) & np.isnan(want))))
    print(case, img.shape, "bad", len(bad))
    for y, x in bad[:6]:
        print("   ", y, x, got[y, x], want[y, x], "row", got[y, max(0,x-3):x+4], want[y, max(0,x-3):x+4])
