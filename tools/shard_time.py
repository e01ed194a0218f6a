"""Sharded densify-step timing only (diagnostics): bench.py's densify_sharded section, N=1."""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

args = types.SimpleNamespace(steps=20, warmup=5, no_cpu=True)
r = bench.bench_densify_sharded(args, 1, 0, torch.device("cuda", 0))
print(json.dumps({"ms": r["ms_per_step"], "split": r["split"], "eligible": r["eligible"]}))
