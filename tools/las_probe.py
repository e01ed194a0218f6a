"""LAS timings (diagnostics): public las_split_batch, the fused cooperative split kernel and the
standalone apply kernel back to back, a CUDA-graph replay of the fused split, at 1M and 100k."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08661_b200 as igs  # noqa: E402
from paper_2603_08661_b200 import _lib  # noqa: E402
from paper_2603_08661_b200.synth import random_cloud_torch  # noqa: E402


def ev_ms(fn, k=10):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


def probe(n):
    dev = torch.device("cuda", 0)
    pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=101, device=dev)
    scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
    mask = torch.ones(n, dtype=torch.bool, device=dev)
    L = _lib.lib()
    c = igs.SplitConstants()
    alpha, la, lg, beta = c.device_constants()
    ws = _lib.workspace(_lib.query_size(L.igs_las_workspace_bytes, n), dev, "las")
    summ = torch.zeros(2, dtype=torch.int64, device=dev)
    m8 = mask.view(torch.uint8)
    fused = lambda: L.igs_las_split(scene._pos.data_ptr(), scene._ls.data_ptr(), scene._rot.data_ptr(),  # noqa: E731
                                    scene._op.data_ptr(), scene._sh.data_ptr(), 48, n, 2 * n,
                                    m8.data_ptr(), alpha, la, lg, beta, ws.data_ptr(), ws.numel(),
                                    summ.data_ptr(), _lib.stream_handle())
    for _ in range(3):
        fused()
    res = {"n": n, "fused_kernel_ms": round(ev_ms(fused), 4)}
    L.igs_las_prepare(m8.data_ptr(), scene._rot.data_ptr(), scene._op.data_ptr(), n, beta,
                      ws.data_ptr(), ws.numel(), summ.data_ptr(), _lib.stream_handle())
    apply = lambda: L.igs_las_apply(scene._pos.data_ptr(), scene._ls.data_ptr(), scene._rot.data_ptr(),  # noqa: E731
                                    scene._op.data_ptr(), scene._sh.data_ptr(), 48, n, 2 * n,
                                    m8.data_ptr(), alpha, la, lg, beta, 0, ws.data_ptr(),
                                    ws.numel(), _lib.stream_handle())
    for _ in range(3):
        apply()
    res["apply_kernel_ms"] = round(ev_ms(apply), 4)
    # CUDA graph of the fused split (the C1 shape of BASELINE configs[0] when n = 100k)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fused()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fused()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    res["fused_graph_ms"] = round(ev_ms(g.replay), 4)
    # the public call (host overhead + one stream sync), restoring the count between calls
    times = []
    for it in range(25):
        scene._set_count(n)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        igs.las_split_batch(scene, mask)
        b.record()
        torch.cuda.synchronize()
        if it >= 5:
            times.append(a.elapsed_time(b))
    res["public_ms"] = round(statistics.median(times), 4)
    return res


print(json.dumps([probe(1_000_000), probe(100_000)]))
