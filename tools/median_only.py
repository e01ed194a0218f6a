"""Median-normalisation-only mode (igs_median_normalize: histogram chunks + collect + apply, no
fused E work) on 200 thinned-map-shaped arrays: time and per-task trace (diagnostics)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import _lib
from paper_2603_08661_b200.synth import synth_views_torch

H, W, B = 822, 1237, 200
views = synth_views_torch(B, H, W, seed=1000, device="cuda")
thin = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
igs.importance_batch(views, out=thin, median=False)
out = torch.empty_like(thin)
flat_in, flat_out = thin.view(B, -1), out.view(B, -1)
for _ in range(3):
    igs.edge_pipeline._median_normalize_batched(flat_in, flat_out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    igs.edge_pipeline._median_normalize_batched(flat_in, flat_out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(json.dumps({"median_only_ms": round(ms, 3), "GB/s_3pass": round(3 * thin.numel() * 8 / ms / 1e6, 1)}))
L = _lib.lib()
cap = 1 << 20
buf = torch.zeros(cap * 4, dtype=torch.int64, device="cuda")
L.igs_debug_edge_trace(buf.data_ptr(), cap, None)
igs.edge_pipeline._median_normalize_batched(flat_in, flat_out)
torch.cuda.synchronize()
n = ctypes.c_int64(0)
L.igs_debug_edge_trace(None, 0, ctypes.byref(n))
rec = buf[: n.value * 4].view(-1, 4).cpu().numpy()
kind = (rec[:, 2].astype(np.uint64) & 0xffffffff).astype(np.int64)
d = rec[:, 1] - rec[:, 0]
print(json.dumps({k: {"n": int((kind == i).sum()), "mean_us": float(d[kind == i].mean() / 1e3) if (kind == i).any() else 0}
                  for i, k in ((1, "H"), (2, "C"), (3, "A"), (4, "NONE"))}))
