"""densify_step latency on 1M (take 5%): polling the pinned results vs a stream sync (diagnostics)."""
import os, statistics, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import las_split as LS
from paper_2603_08661_b200.synth import random_cloud_torch, random_stats
dev = torch.device("cuda", 0)
n = 1_000_000
pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=101, device=dev)
scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
pristine = {k: getattr(scene, k)[:n].clone() for k in ("_pos", "_ls", "_op")}
grad, edge = random_stats(n, seed=7)
def run(reps=25):
    ts = []
    for it in range(reps):
        for k, v in pristine.items():
            getattr(scene, k)[:n].copy_(v)
        scene._set_count(n)
        stats = igs.DensifyStats(n, device=dev)
        stats._grad_sum.copy_(torch.from_numpy(grad))
        stats._accum_count = 1
        stats.set_edge_score(edge)
        cfg = igs.DensifyConfig(budget=2 * n)
        torch.cuda.synchronize()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ev = igs.densify_step(scene, stats, cfg, 2000)
        c.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(a.elapsed_time(c))
    return round(statistics.median(ts), 4), ev.split
res = {"poll": run()}
ws, ww = LS.wait_summary, LS.wait_word
LS.wait_summary = lambda d, b: LS.sync(d)
LS.wait_word = lambda d, b, i: None
res["sync"] = run()
LS.wait_summary, LS.wait_word = ws, ww
res["poll2"] = run()
print(json.dumps(res))
# kernel timeline of one step in each mode (torch.profiler)
from torch.profiler import profile, ProfilerActivity
def one():
    for k, v in pristine.items():
        getattr(scene, k)[:n].copy_(v)
    scene._set_count(n)
    stats = igs.DensifyStats(n, device=dev)
    stats._grad_sum.copy_(torch.from_numpy(grad))
    stats._accum_count = 1
    stats.set_edge_score(edge)
    cfg = igs.DensifyConfig(budget=2 * n)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        igs.densify_step(scene, stats, cfg, 2000)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t0 = min(e.time_range.start for e in evs)
    return [(e.name[:40], round(e.time_range.start - t0, 1), round(e.time_range.elapsed_us(), 1)) for e in sorted(evs, key=lambda e: e.time_range.start)]
for mode in ("poll", "sync"):
    if mode == "sync":
        LS.wait_summary = lambda d, b: LS.sync(d)
        LS.wait_word = lambda d, b, i: None
    one()
    print(mode, json.dumps(one()))
