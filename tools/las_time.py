"""LAS timing only (diagnostics): bench.py's las section on cuda:0."""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

args = types.SimpleNamespace(steps=20, warmup=5, no_cpu=True)
peak, src = bench.peaks()
r = bench.bench_las(args, 1, torch.device("cuda", 0), peak, src)
print(json.dumps({"kernel_ms": r["roofline"]["kernel_ms"], "frac": r["roofline"]["frac"],
                  "split_device_ms": r["roofline"]["split_device_ms"],
                  "las_ms": r["ms_per_step"], "densify_ms": r["densify_step"]["ms"]}))
