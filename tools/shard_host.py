"""Host time per stage of one sharded densify step at N=1 (diagnostics): the sharded module's
stage functions wrapped with perf_counter spans (~1 us of wrapper overhead each)."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08661_b200 as igs  # noqa: E402
from paper_2603_08661_b200 import sharded, _lib  # noqa: E402
from paper_2603_08661_b200.synth import random_cloud_torch, random_stats  # noqa: E402

n = 6_000_000
dev = torch.device("cuda", 0)
pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=301, device=dev)
scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
pristine = {k: getattr(scene, k)[:n].clone() for k in ("_pos", "_ls", "_op")}
grad, edge = random_stats(n, seed=17)
grad_t = torch.from_numpy(grad).to(dev)
comm = sharded.Comm()
caps = sharded.global_counts(scene, comm)
cfg = igs.DensifyConfig(budget=2 * n)
spans = collections.defaultdict(list)


def wrap(obj, name, label):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter_ns()
        r = f(*a, **k)
        spans[label].append((t, time.perf_counter_ns()))
        return r
    setattr(obj, name, g)


for nm in ("_publish", "_split_guarded", "_read", "attach", "_reserve", "_take_cap_global",
           "_protocol"):
    wrap(sharded, nm, nm)
for nm in ("keys", "boundary", "finalize"):
    wrap(sharded.CudaShardOps, nm, "ops." + nm)
wrap(igs.DensifyStats, "reset", "stats.reset")

for it in range(8):
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
    spans.clear()
    t0 = time.perf_counter_ns()
    sharded.densify_step_sharded(scene, st, cfg, 2000, comm, caps=caps)
    t1 = time.perf_counter_ns()
    torch.cuda.synchronize()
    t2 = time.perf_counter_ns()
rows = sorted((s[0], s[1], k) for k, v in spans.items() for s in v)
for a, b, k in rows:
    print(f"{(a - t0) / 1e3:8.1f} .. {(b - t0) / 1e3:8.1f} us  {k}")
print(f"call returns at {(t1 - t0) / 1e3:.1f} us, stream idle at {(t2 - t0) / 1e3:.1f} us")
