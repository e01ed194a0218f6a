"""Edge kernel time vs L2 persisting set-aside (igs_l2_set_aside) and ahead (diagnostics)."""
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
maxp = ctypes.c_int(0)
for mb in [int(x) for x in os.environ.get("SETASIDE", "0 32 64 96").split()]:
    g = ctypes.c_size_t(0)
    L.igs_l2_set_aside(mb << 20, ctypes.byref(g))
    for _ in range(3):
        igs.importance_batch(views, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        igs.importance_batch(views, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"setaside_MB": mb, "granted_MB": g.value >> 20, "ahead": os.environ.get("IGS_AHEAD"),
                      "bh": os.environ.get("IGS_BAND_H"), "ms": round(ms, 3),
                      "GPix/s": round(B * H * W / ms / 1e6, 2)}))
