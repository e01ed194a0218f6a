import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, paper_2603_08661_b200 as igs
from paper_2603_08661_b200.synth import synth_views_torch
H, W = 822, 1237
for B in (1, 4):
    v = synth_views_torch(B, H, W, seed=3000, device="cuda")
    out = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
    for _ in range(3): igs.importance_batch(v, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): igs.importance_batch(v, out=out)
    b.record(); torch.cuda.synchronize()
    print(B, round(a.elapsed_time(b) / 20, 4), end="  ")
print()
