"""configs[0] LAS latency pieces (diagnostics): CUDA-event time of the public call and of the
launches alone, host time of each piece, on 100k SH3 Gaussians all masked."""
import json, os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import las_split as LS
from paper_2603_08661_b200.synth import random_cloud_torch
dev = torch.device("cuda", 0)
n = 100_000
pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=7, device=dev)
scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
mask = torch.ones(n, dtype=torch.bool, device=dev)
c = igs.SplitConstants()
pristine = {k: getattr(scene, k)[:n].clone() for k in ("_pos", "_ls", "_op")}
def reset():
    for k, v in pristine.items():
        getattr(scene, k)[:n].copy_(v)
    scene._set_count(n)
    torch.cuda.synchronize()
def ev(fn, reps=30):
    ts, hs = [], []
    for it in range(reps):
        reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); t0 = time.perf_counter()
        fn()
        t1 = time.perf_counter(); b.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(b) * 1e3); hs.append((t1 - t0) * 1e6)
    return round(statistics.median(ts), 1), round(statistics.median(hs), 1)
buf, view = LS.pinned_summary(dev)
res = {}
res["public_gpu_us, host_us"] = ev(lambda: igs.las_split_batch(scene, mask, c))
res["split_async_gpu_us, host_us"] = ev(lambda: LS.split_async(scene, mask, c, summary=buf))
empty = torch.empty(1, device=dev)
res["torch_fill_gpu_us, host_us"] = ev(lambda: empty.fill_(1.0))
print(json.dumps(res))
# host time of the bare C call (arguments precomputed)
from paper_2603_08661_b200 import _lib
L = _lib.lib()
m = LS._mask_tensor(mask, n, dev)
nbytes = _lib.query_size(L.igs_las_workspace_bytes, n)
ws = _lib.workspace(nbytes, dev, "las")
alpha, la, lg, beta = c.device_constants()
st = _lib.stream_handle(dev)
p5 = LS._column_ptrs(scene)
args = (*p5, scene._sh.shape[1] * 3, n, scene.capacity, m.data_ptr(), alpha, la, lg, beta,
        ws.data_ptr(), ws.numel(), buf.data_ptr(), st)
def bare():
    L.igs_las_split(*args)
res2 = {"bare_C_call_gpu_us, host_us": ev(bare)}
def bare_sparse():
    L.igs_las_split_sparse(*args)
res2["bare_sparse_gpu_us, host_us"] = ev(bare_sparse)
print(json.dumps(res2))
