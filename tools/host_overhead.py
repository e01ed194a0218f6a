"""Host-side overhead of the public LAS call (diagnostics): per-call microseconds of its pieces."""
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


def us(fn, k=2000):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t) / k * 1e6, 2)


n = 1000
dev = torch.device("cuda", 0)
pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=101, device=dev)
scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
mask = torch.zeros(n, dtype=torch.bool, device=dev)
# all-false mask: the kernel runs its pre-pass and writes nothing (host cost only)
L = _lib.lib()
c = igs.SplitConstants()
buf, view = LS.pinned_summary(dev)
s = torch.cuda.current_stream()
res = {
    "ctypes_abi_version": us(lambda: L.igs_abi_version()),
    "torch_current_stream": us(lambda: torch.cuda.current_stream(dev)),
    "stream_handle": us(lambda: _lib.stream_handle()),
    "lib_check": us(lambda: _lib.lib()),
    "mask_tensor": us(lambda: LS._mask_tensor(mask, n, dev)),
    "pinned_summary": us(lambda: LS.pinned_summary(dev)),
    "split_async_only": us(lambda: LS.split_async(scene, mask, c, summary=buf), 500),
    "sync_idle_stream": us(lambda: s.synchronize()),
    "split_async_plus_sync": us(lambda: (LS.split_async(scene, mask, c, summary=buf), s.synchronize()), 500),
}


def public():
    scene._set_count(n)
    igs.las_split_batch(scene, mask)


res["las_split_batch"] = us(public, 500)
alpha, la, lg, beta = c.device_constants()
ws = _lib.workspace(_lib.query_size(L.igs_las_workspace_bytes, n), dev, "las")
m8 = mask.view(torch.uint8)
st = _lib.stream_handle()
args = (scene._pos.data_ptr(), scene._ls.data_ptr(), scene._rot.data_ptr(), scene._op.data_ptr(),
        scene._sh.data_ptr(), 48, n, 2 * n, m8.data_ptr(), alpha, la, lg, beta, ws.data_ptr(),
        ws.numel(), buf.data_ptr(), st)
res["cabi_las_split"] = us(lambda: L.igs_las_split(*args), 500)
res["cabi_las_prepare"] = us(lambda: L.igs_las_prepare(m8.data_ptr(), scene._rot.data_ptr(),
                                                     scene._op.data_ptr(), n, beta, ws.data_ptr(),
                                                     ws.numel(), buf.data_ptr(), st), 500)
aargs = args[:13] + (0,) + args[13:15] + (st,)
res["cabi_las_apply"] = us(lambda: L.igs_las_apply(*aargs), 500)
print(json.dumps(res))
