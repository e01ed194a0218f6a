"""Per-task timeline of one fused edge launch (diagnostics)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import _lib
from paper_2603_08661_b200.synth import synth_views_torch

H, W, B = 822, 1237, int(os.environ.get("VIEWS", "200"))
views = synth_views_torch(B, H, W, seed=1000, device="cuda")
out = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
for _ in range(3):
    igs.importance_batch(views, out=out)
L = _lib.lib()
cap = 1 << 20
buf = torch.zeros(cap * 4, dtype=torch.int64, device="cuda")
L.igs_debug_edge_trace(buf.data_ptr(), cap, None)
igs.importance_batch(views, out=out)
torch.cuda.synchronize()
n = ctypes.c_int64(0)
L.igs_debug_edge_trace(None, 0, ctypes.byref(n))
rec = buf[: n.value * 4].view(-1, 4).cpu().numpy()
t0, t1 = rec[:, 0].astype(np.int64), rec[:, 1].astype(np.int64)
kvi = rec[:, 2].astype(np.uint64)
kind = (kvi & 0xffffffff).astype(np.int64)
view = (kvi >> 32).astype(np.int64)
base = t0.min()
span = t1.max() - base
names = {1: "E", 2: "C", 3: "A", 4: "NONE"}
res = {"records": int(n.value), "span_us": span / 1e3}
for k, nm in names.items():
    m = kind == k
    d = (t1 - t0)[m]
    res[nm] = {"n": int(m.sum()), "busy_us_total": float(d.sum() / 1e3),
               "mean_us": float(d.mean() / 1e3) if m.any() else 0}
# fronts: when each view's E finished vs A finished
e_end = np.zeros(B); a_end = np.zeros(B); e_beg = np.full(B, np.inf); c_end = np.zeros(B)
for k_, v_, s_, e_ in zip(kind, view, t0 - base, t1 - base):
    if k_ == 1:
        e_end[v_] = max(e_end[v_], e_); e_beg[v_] = min(e_beg[v_], s_)
    if k_ == 2:
        c_end[v_] = max(c_end[v_], e_)
    if k_ == 3:
        a_end[v_] = max(a_end[v_], e_)
lat = (a_end - e_end) / 1e3
res["view_E_span_us_mean"] = float(((e_end - e_beg) / 1e3).mean())
res["E_end_to_C_end_us_mean"] = float(((c_end - e_end) / 1e3).mean())
res["E_end_to_A_end_us_mean"] = float(lat.mean())
res["E_end_to_A_end_us_max"] = float(lat.max())
res["slots_x_span_us"] = float(span / 1e3 * len(np.unique(rec[:, 3] >> 32)) )
print(json.dumps(res, indent=1))
np.save("gpurun_out/edge_trace.npy", rec)
