"""Per-phase time of the fused edge kernel's band sub-steps.  Needs a library built with
-DIGS_PHASE_PROF (IGS_LIB=...): thread 0's barrier-to-barrier times, summed over blocks."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import _lib
from paper_2603_08661_b200.synth import synth_views_torch

H, W, B = 822, 1237, 200
views = synth_views_torch(B, H, W, seed=1000, device="cuda")
out = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
L = _lib.lib()
buf = (ctypes.c_uint64 * 8)()
for name, kw in (("full", {}), ("no_median", {"median": False})):
    for _ in range(2):
        igs.importance_batch(views, out=out, **kw)
    torch.cuda.synchronize()
    L.igs_debug_edge_phases(buf, 1)
    igs.importance_batch(views, out=out, **kw)
    torch.cuda.synchronize()
    L.igs_debug_edge_phases(buf, 1)
    tot = sum(buf[:7])
    print(name, json.dumps({k: round(100 * buf[i] / tot, 1) for i, k in
                            enumerate(("unused", "blur", "sobel", "decide",
                                       "finish+next gray", "blur_last+claim", "prologue"))}),
          "block-ms", round(tot / 1e6, 1))
