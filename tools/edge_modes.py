"""Time the fused edge kernel in its modes (diagnostics, not the headline bench)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200.synth import synth_views_torch

H, W, B = 822, 1237, int(os.environ.get("VIEWS", "200"))
views = synth_views_torch(B, H, W, seed=1000, device="cuda")
out = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
res = {}
for name, kw in (("full", {}), ("no_median", {"median": False}),
                 ("no_nms_no_median", {"nms": False, "median": False})):
    for _ in range(3):
        igs.importance_batch(views, out=out, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 20
    for _ in range(n):
        igs.importance_batch(views, out=out, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    res[name] = {"ms": round(ms, 3), "GPix/s": round(B * H * W / ms / 1e6, 2)}
print(json.dumps(res))
