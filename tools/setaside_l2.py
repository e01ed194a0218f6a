"""Edge kernel (full mode) with a persisting-L2 set-aside: time (diagnostics); run under ncu
for DRAM bytes.  SETASIDE_MB env (default 79)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import _lib
from paper_2603_08661_b200.synth import synth_views_torch

H, W, B = 822, 1237, 200
views = synth_views_torch(B, H, W, seed=1000, device="cuda")
out = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
g = ctypes.c_size_t(0)
_lib.lib().igs_l2_set_aside(int(os.environ.get("SETASIDE_MB", "79")) << 20, ctypes.byref(g))
for _ in range(4):
    igs.importance_batch(views, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    igs.importance_batch(views, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"granted_MB": g.value >> 20, "ms": round(ms, 3), "GPix/s": round(B * H * W / ms / 1e6, 2)}))
