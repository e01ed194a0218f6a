"""Timeline of one sharded densify step at N=1 (diagnostics): torch.profiler (CUPTI) kernel
and memcpy spans, with the gaps between them (host work the GPU waits for)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2603_08661_b200 as igs  # noqa: E402
from paper_2603_08661_b200 import sharded  # noqa: E402
from paper_2603_08661_b200.synth import random_cloud_torch, random_stats  # noqa: E402

n = int(os.environ.get("N", "6000000"))
dev = torch.device("cuda", 0)
pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=301, device=dev)
scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
pristine = {k: getattr(scene, k)[:n].clone() for k in ("_pos", "_ls", "_op")}
grad, edge = random_stats(n, seed=17)
grad_t = torch.from_numpy(grad).to(dev)
comm = sharded.Comm()
caps = sharded.global_counts(scene, comm)
cfg = igs.DensifyConfig(budget=2 * n)


def step():
    for k, v in pristine.items():
        getattr(scene, k)[:n].copy_(v)
    scene._set_count(n)
    sharded.detach(scene)
    sharded.attach(scene, comm, caps)
    st = igs.DensifyStats(n, device=dev)
    st._grad_sum.copy_(grad_t)
    st._accum_count = 1
    st.set_edge_score(edge)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("step")
    sharded.densify_step_sharded(scene, st, cfg, 2000, comm, caps=caps)
    torch.cuda.nvtx.range_pop()


for _ in range(3):
    step()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
# only the step's kernels: after the last pre-step synchronize (the largest gap)
t0 = None
rows = []
for e in ev:
    rows.append((e.time_range.start, e.time_range.end, e.name[:60]))
starts = [r[0] for r in rows]
# find the first kernel of the step: after the biggest idle gap
gaps = [(rows[i][0] - rows[i - 1][1], i) for i in range(1, len(rows))]
first = max(gaps)[1] if gaps else 0
prev = rows[first][0]
tot0 = rows[first][0]
for s, e, name in rows[first:]:
    print(f"+{(s - tot0):8.1f} us  gap {s - prev:7.1f}  dur {e - s:7.1f}  {name}")
    prev = e
print(f"device span {rows[-1][1] - tot0:.1f} us")

# host-side view of the step: CPU op spans from the same profile
cpu = [e for e in prof.events() if e.device_type.name == "CPU"]
cpu.sort(key=lambda e: e.time_range.start)
t0 = cpu[0].time_range.start if cpu else 0
for e in cpu:
    d = e.time_range.end - e.time_range.start
    if d > 4.0:
        print(f"cpu +{e.time_range.start - t0:8.1f} us dur {d:7.1f}  {e.name[:70]}")
