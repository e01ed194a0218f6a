"""configs[0] edge latency (one 1237x822 view) under the current IGS_* settings (diagnostics)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200.synth import synth_views_torch
v = synth_views_torch(1, 822, 1237, seed=3000, device="cuda")
out = torch.empty((1, 822, 1237), dtype=torch.float64, device="cuda")
for _ in range(5):
    igs.importance_batch(v, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    igs.importance_batch(v, out=out)
b.record()
torch.cuda.synchronize()
print(json.dumps({"band_h": os.environ.get("IGS_BAND_H"), "chunk": os.environ.get("IGS_CHUNK"),
                  "ms": round(a.elapsed_time(b) / 50, 4)}))
