"""sample_scores / accumulate_position_grads kernel timing only (diagnostics): bench.py's aux."""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

args = types.SimpleNamespace(steps=10, warmup=3, no_cpu=True)
peak, _ = bench.peaks()
r = bench.bench_aux(args, 1, torch.device("cuda", 0), peak)
print(json.dumps({k: (v["kernel_ms"], v["roofline"]["frac"]) for k, v in r.items() if k != "config"}))
