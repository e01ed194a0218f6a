"""L2 residency experiment: edge kernel time with/without a persisting set-aside."""
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
res = {}
props = torch.cuda.get_device_properties(0)
res["l2_bytes"] = props.L2_cache_size
for mb in [int(x) for x in os.environ.get("SETASIDE", "0,32,64,96").split(",")]:
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
    res[f"setaside_{mb}MB(granted {g.value >> 20}MB)"] = round(e0.elapsed_time(e1) / 10, 3)
print(json.dumps(res))
