"""Host-side cost of each step of the public las_split_batch at configs[0] size (diagnostics):
microseconds per call of each piece, measured in a loop of calls."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08661_b200 as igs  # noqa: E402
from paper_2603_08661_b200 import _lib  # noqa: E402
from paper_2603_08661_b200 import las_split as LS  # noqa: E402
from paper_2603_08661_b200.synth import random_cloud_torch  # noqa: E402

n = 100_000
dev = torch.device("cuda", 0)
pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=101, device=dev)
scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
mask = torch.zeros(n, dtype=torch.bool, device=dev)   # nothing splits: host cost + kernels
c = igs.SplitConstants()
L = _lib.lib()


def us(fn, k=3000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t) / k * 1e6, 2)


buf, view = LS.pinned_summary(dev)
res = {
    "mask_tensor": us(lambda: LS._mask_tensor(mask, n, dev)),
    "query_size": us(lambda: _lib.query_size(L.igs_las_workspace_bytes, n)),
    "workspace": us(lambda: _lib.workspace(1 << 20, dev, "las")),
    "device_constants": us(lambda: c.device_constants()),
    "stream_handle": us(lambda: _lib.stream_handle(dev)),
    "column_ptrs": us(lambda: LS._column_ptrs(scene)),
    "pinned_summary": us(lambda: LS.pinned_summary(dev)),
    "split_async": us(lambda: LS.split_async(scene, mask, c, summary=buf), 1000),
    "sync_idle": us(lambda: LS.sync(dev)),
    "public_call": us(lambda: igs.las_split_batch(scene, mask), 1000),
}
print(json.dumps(res))
