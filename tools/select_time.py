"""Single-GPU select timing (diagnostics): igs_select_candidates at 1M and 6M, back to back."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_08661_b200 as igs  # noqa: E402

res = {}
for n in (1_000_000, 6_000_000):
    rng = np.random.default_rng(7)
    st = igs.DensifyStats(n)
    igs.accumulate_grads(st, rng.exponential(2e-4, n))
    st.set_edge_score(rng.random(n))
    cfg = igs.DensifyConfig(budget=2 * n)
    for _ in range(3):
        igs.select_candidates(st, cfg, 2000, n)
    torch.cuda.synchronize()
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        igs.select_candidates(st, cfg, 2000, n)
    c.record()
    torch.cuda.synchronize()
    res[n] = round(a.elapsed_time(c) / 10, 4)
print(json.dumps(res))
