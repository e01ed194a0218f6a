"""Benchmark of the B200 densification hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (N=1 workload = BASELINE.json configs[1]): edge-importance maps + per-view
median normalisation over 200 synthetic 1237x822 RGB float64 views per GPU
("edge-map MPix/s").  One step = one importance_batch() over the 200 resident views
(one fused persistent kernel launch).  Inputs (4.9 GB) are far larger than L2, so
no flush is needed between steps.  Secondary object "las": Long-Axis-Split of a 1M-
Gaussian SH-degree-3 cloud (configs[2], all-masked bandwidth case) plus the full
densify_step (select 50k of 1M + LAS).

Multi-GPU (torchrun, one rank per GPU): views shard per GPU (weak scaling, no
collective on the data path); value = all ranks' pixels / max-over-ranks time.

--impl reference: the reference's CPU path on this host -- the unmodified
splitkit.edge_pipeline.importance_pipeline installed in baseline/_ref (else the oracle
restatement oracle/edge.py) over a pool of all host cores, one view per process per step;
rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W = 822, 1237
PX = H * W
VIEWS = 200
BYTES_PER_PX_F64 = 24 + 8          # f64 RGB in + f64 map out
LAS_N = 1_000_000
LAS_BYTES_PER_SPLIT = 236 + 28 + 236  # read record, in-place parent, appended child
METRIC = "edge-map MPix/s"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """DRAM bytes per unit from the committed ncu capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms while active."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.idx = device_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    """One process per GPU (torchrun env).  IGS_DIST_BACKEND=gloo (plumbing test only) lets
    several ranks share one GPU: the device is LOCAL_RANK modulo the visible GPUs."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        backend = os.environ.get("IGS_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ CPU reference
REF_PATH = os.path.join(ROOT, "baseline", "_ref")  # the unmodified splitkit


def ref_kind():
    """"reference" when the unmodified splitkit is installed in baseline/_ref (it travels to
    the GPU box with the snapshot), else "port" (the oracle restatement)."""
    return "reference" if os.path.isdir(os.path.join(REF_PATH, "splitkit")) else "port"


def ref_edge_fn():
    if ref_kind() == "reference":
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        from splitkit.edge_pipeline import importance_pipeline
        return importance_pipeline
    from oracle import edge as OE
    return OE.importance_pipeline


_CPU_VIEW = None
_CPU_FN = None


def _cpu_init(seed):
    global _CPU_VIEW, _CPU_FN
    from paper_2603_08661_b200.synth import synth_view
    _CPU_VIEW = synth_view(H, W, seed + os.getpid() % 97)
    _CPU_FN = ref_edge_fn()


def _cpu_task(_):
    t0 = time.perf_counter()
    _CPU_FN(_CPU_VIEW)
    return time.perf_counter() - t0


def cpu_edge_rate(steps, warmup, procs=None):
    """Reference edge pipeline over a process pool of all host cores (one 1237x822 view per
    process per step) -> (MPix/s, processes, seconds per step)."""
    import multiprocessing as mp
    procs = procs or len(os.sched_getaffinity(0))
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs, initializer=_cpu_init, initargs=(1000,)) as pool:
        for _ in range(warmup):
            pool.map(_cpu_task, range(procs), chunksize=1)
        t0 = time.perf_counter()
        for _ in range(steps):
            pool.map(_cpu_task, range(procs), chunksize=1)
        wall = time.perf_counter() - t0
    return steps * procs * PX / wall / 1e6, procs, wall / steps


def cpu_las_rate(n=200_000):
    """Reference las_split_batch, all masked, 1 core.  The reference Scene3 holds 3-float
    colours (core.py:172), so its LAS moves 56 B per record, not the 236 B SH3 record."""
    import numpy as np
    from paper_2603_08661_b200.synth import random_cloud
    pos, ls, q, o, sh = random_cloud(n, 16, seed=101)
    mask = np.ones(n, bool)
    reps = 3
    if ref_kind() == "reference":
        if REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        from splitkit.core import Scene3
        from splitkit.las_split import las_split_batch
        scenes = [Scene3(pos, ls, q, o, sh[:, 0, :], capacity=2 * n) for _ in range(reps + 1)]
        las_split_batch(scenes[0], mask)
        t0 = time.perf_counter()
        for k in range(reps):
            las_split_batch(scenes[k + 1], mask)
        return n * reps / (time.perf_counter() - t0), "reference", \
            f"{reps} x {n // 1000}k all-masked, splitkit.las_split_batch (colour-only records)"
    from oracle import las as OL
    d = {"positions": pos, "log_scales": ls, "rotations": q, "opacity_logits": o, "sh": sh,
         "capacity": 2 * n}
    OL.las_split_batch(d, mask)
    t0 = time.perf_counter()
    for _ in range(reps):
        OL.las_split_batch(d, mask)
    return n * reps / (time.perf_counter() - t0), "port", \
        f"{reps} x {n // 1000}k all-masked, SH degree 3, oracle/las.py"


def edge_config(world):
    """The headline line's config, shared by both arms (the driver compares them key by key)."""
    return {"workload": "200 x 1237x822 RGB f64 views per GPU: gray+blur+Sobel+NMS+"
                        "median normalisation (BASELINE.json configs[1])",
            "views_per_gpu": VIEWS, "height": H, "width": W, "io": "f64 in / f64 out",
            "l2": "inputs 4.9 GB per GPU >> 126 MB L2 (no flush needed)",
            "parallelism": f"views sharded, {world} GPU(s), no data-path collective"}


def run_reference(args, world, rank):
    """The reference arm: the unmodified splitkit importance_pipeline (baseline/_ref, else the
    oracle port) on all host cores, with the same --steps / --warmup and config as the GPU arm;
    each step is a bounded sample of the workload (one 1237x822 view per host process), and
    the metric is the same per-pixel throughput."""
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    rate, procs, sec = cpu_edge_rate(steps, warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(rate, 3), "unit": "MPix/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": edge_config(world),
        "cpu_baseline": {"value": round(rate, 3), "unit": "MPix/s", "cores": procs,
                         "kind": ref_kind(),
                         "sample": f"{procs} views per step (1 per process), "
                                   + ("splitkit.edge_pipeline.importance_pipeline (baseline/_ref)"
                                      if ref_kind() == "reference" else
                                      "oracle/edge.py restatement of splitkit.edge_pipeline")},
        "e2e": {"value": round(rate, 3), "unit": "MPix/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU (ours)
def run_ours(args, world, rank, local):
    import torch

    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200.synth import synth_views_torch

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    peak, peak_src = peaks()
    views = synth_views_torch(VIEWS, H, W, seed=1000 + 17 * rank, device=dev)
    out = torch.empty((VIEWS, H, W), dtype=torch.float64, device=dev)
    for _ in range(args.warmup):
        igs.importance_batch(views, out=out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            igs.importance_batch(views, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms, world)
    check = None if args.no_check else check_sample(views, out)
    value = world * VIEWS * PX / (ms * 1e-3) / 1e6
    algo_bytes = VIEWS * PX * BYTES_PER_PX_F64
    achieved = algo_bytes / (ms * 1e-3) / 1e9
    traffic = ncu_traffic().get("edge_persistent_kernel_bytes_per_px")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "MPix/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": edge_config(world),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": (round(traffic * VIEWS * PX) if traffic else None),
                     "kernel": "edge_persistent_kernel", "algorithmic_bytes_per_px": 32,
                     "peak_source": peak_src,
                     "frac_datasheet_8TBps": round(achieved / 8000.0, 4),
                     "fp64_pipe_active_pct": ncu_traffic().get("edge_fp64_pipe_active_pct"),
                     "issue_active_pct": ncu_traffic().get("edge_issue_active_pct"),
                     "note": "the kernel is issue/latency-bound (FP64 blur + integer NMS work); "
                             "fp64 / issue figures from the committed ncu --set full capture"},
        "per_gpu_value": round(value / world, 3),
        "check": check,
        "clocks": clk.summary(),
        "gpu_launches": args.steps,
    }
    if not args.no_e2e:
        line["e2e"] = e2e_edge(args, world, dev)
    def section(name, fn, *a):
        """A secondary measurement: its failure is recorded in the line, never fatal to the
        headline (every rank runs the same sections, so collectives stay matched)."""
        try:
            line[name] = fn(*a)
        except Exception as exc:  # pragma: no cover - reported, not hidden
            line[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if not args.no_uhd:
        section("edge_uhd", bench_uhd, args, world, dev, peak)
        section("edge_f32_input", bench_f32_input, args, world, dev, peak)
    if not args.no_las:
        section("las", bench_las, args, world, dev, peak, peak_src)
        section("densify_sharded", bench_densify_sharded, args, world, rank, dev)
        section("aux", bench_aux, args, world, dev, peak)
        section("c1", bench_c1, args, world, dev)
        if rank == 0:
            section("scene_io", bench_scene_io, args, dev)
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, procs, _ = cpu_edge_rate(2, 1)
        line["cpu_baseline"] = {"value": round(rate, 3), "unit": "MPix/s", "cores": procs,
                                "kind": ref_kind(),
                                "sample": f"2x{procs} views (1 per process per step), "
                                          + ("splitkit importance_pipeline (baseline/_ref)"
                                             if ref_kind() == "reference" else "oracle/edge.py")
                                          + " on the host cores"}
    if rank == 0:
        print(json.dumps(line), flush=True)


CHECK_VIEWS = (0, 16, 99, 199)


def check_sample(views, out):
    """The timed launch's own output for a sample of views (both sides of the 16-slot ring's
    wraps) against the CPU path the cpu_baseline leg times (the unmodified reference from
    baseline/_ref, else the oracle restatement) on the same views, outside the timed region:
    bit-exact or the line says so."""
    import numpy as np
    fn = ref_edge_fn()
    res = {}
    for v in CHECK_VIEWS:
        want = fn(views[v].cpu().numpy())
        res[str(v)] = int(np.count_nonzero(out[v].cpu().numpy() != want))
    return {"views": list(CHECK_VIEWS), "differing_pixels": res,
            "bit_exact": all(n == 0 for n in res.values()),
            "against": ("splitkit.edge_pipeline.importance_pipeline (baseline/_ref)"
                        if ref_kind() == "reference" else "oracle/edge.py")}


def e2e_edge(args, world, dev):
    """Public API with host buffers: pinned (B,H,W,3) f64 in, pinned (B,H,W) f64 out; the H2D
    of the inputs and the D2H of the maps are inside the timed region, every step."""
    import torch

    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200.synth import synth_views_torch
    host_in = synth_views_torch(VIEWS, H, W, seed=2000, device=dev).cpu().pin_memory()
    host_out = torch.empty((VIEWS, H, W), dtype=torch.float64).pin_memory()
    steps = max(3, min(args.steps, 20))
    for _ in range(2):
        igs.importance_batch(host_in, out=host_out)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        igs.importance_batch(host_in, out=host_out)   # returns after the D2H has landed
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / steps
    barrier(world)
    sec = max_over_ranks(sec, world)
    return {"value": round(world * VIEWS * PX / sec / 1e6, 3), "unit": "MPix/s",
            "h2d_bytes_per_step": VIEWS * PX * 24, "d2h_bytes_per_step": VIEWS * PX * 8,
            "ms_per_step": round(sec * 1e3, 3), "steps": steps,
            "h2d_GBps": round(VIEWS * PX * 24 / sec / 1e9, 1),
            "bound": "PCIe host->device copy of the float64 views (the kernel takes ~4% of the step)",
            "api": "importance_batch(pinned host views, out=pinned host maps), 8-view chunks "
                   "with H2D / kernel / D2H overlapped on three streams"}


def bench_f32_input(args, world, dev, peak):
    """SURVEY.md 8(d)'s float32-input variant: the same 200 views stored as float32 (12 B/px in,
    float64 maps out: 20 B/px). The reference converts to float64 first (edge_pipeline.py:133),
    so the maps are identical to the float64 run on the converted values. Device-resident, plus
    the end-to-end form with pinned host buffers (8 B/px less over PCIe)."""
    import torch

    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200.synth import synth_views_torch
    views = synth_views_torch(VIEWS, H, W, seed=1000, device=dev).float()
    out = torch.empty((VIEWS, H, W), dtype=torch.float64, device=dev)
    for _ in range(2):
        igs.importance_batch(views, out=out)
    steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        igs.importance_batch(views, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
    achieved = VIEWS * PX * 20 / (ms * 1e-3) / 1e9
    host_in = views.cpu().pin_memory()
    del views
    host_out = torch.empty((VIEWS, H, W), dtype=torch.float64).pin_memory()
    for _ in range(1):
        igs.importance_batch(host_in, out=host_out)
    torch.cuda.synchronize()
    esteps = max(2, min(args.steps, 4))
    t0 = time.perf_counter()
    for _ in range(esteps):
        igs.importance_batch(host_in, out=host_out)
    torch.cuda.synchronize()
    sec = max_over_ranks((time.perf_counter() - t0) / esteps, world)
    del out
    torch.cuda.empty_cache()
    return {"metric": "edge-map MPix/s", "value": round(world * VIEWS * PX / (ms * 1e-3) / 1e6, 3),
            "unit": "MPix/s", "ms_per_step": round(ms, 4), "steps": steps, "dtype_in": "f32",
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "algorithmic_bytes_per_px": 20},
            "e2e": {"value": round(world * VIEWS * PX / sec / 1e6, 3), "unit": "MPix/s",
                    "h2d_bytes_per_step": VIEWS * PX * 12, "d2h_bytes_per_step": VIEWS * PX * 8,
                    "ms_per_step": round(sec * 1e3, 3)},
            "config": {"workload": "the headline's 200 x 1237x822 views as float32 input"}}


def bench_aux(args, world, dev, peak):
    """SURVEY.md 8(f) rows 1-2 at the configs[3] cloud size (6M primitives), kernels timed
    back to back through the C ABI between CUDA events:
    sample_scores   bilinear samples of 8 resident 1237x822 maps, one view index per point:
                    16 B position + 4 B view + 4 x 8 B taps + 8 B score = 60 B per point
    accumulate_position_grads   grad_sum += hypot(g) in float64: 16 B + 8 B + 8 B = 32 B"""
    import torch

    from paper_2603_08661_b200 import _lib
    L = _lib.lib()
    n, nm = DENSIFY_N, 8
    g = torch.Generator(device=dev).manual_seed(3)
    maps = torch.rand((nm, H, W), dtype=torch.float64, device=dev, generator=g)
    pos = torch.stack([torch.rand(n, dtype=torch.float64, device=dev, generator=g) * (W - 1),
                       torch.rand(n, dtype=torch.float64, device=dev, generator=g) * (H - 1)], 1)
    view = torch.randint(0, nm, (n,), dtype=torch.int32, device=dev, generator=g)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    grads = torch.randn((n, 2), dtype=torch.float64, device=dev, generator=g) * 1e-4
    gsum = torch.zeros(n, dtype=torch.float64, device=dev)
    sh = _lib.stream_handle(dev)

    def timed(fn, k=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        c.record()
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(c) / k, world)

    ms_s = timed(lambda: L.igs_sample_scores(maps.data_ptr(), nm, H, W, pos.data_ptr(),
                                             view.data_ptr(), n, out.data_ptr(),
                                             flags.data_ptr(), sh))
    ms_g = timed(lambda: L.igs_accumulate_grad_norms(gsum.data_ptr(), grads.data_ptr(),
                                                     _lib.IGS_F64, n, sh))
    del maps, pos, view, out, grads, gsum
    torch.cuda.empty_cache()

    def line(ms, bpu, what):
        ach = n * bpu / (ms * 1e-3) / 1e9
        return {"metric": f"{what} per s", "value": round(world * n / (ms * 1e-3), 1),
                "kernel_ms": round(ms, 4),
                "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                             "unit": "GB/s", "frac": round(ach / peak, 4),
                             "algorithmic_bytes_per_unit": bpu}}
    return {"sample_scores": line(ms_s, 60, "points"),
            "accumulate_position_grads": line(ms_g, 32, "primitives"),
            "config": {"workload": "6M points / primitives (configs[3] size); 8 resident maps",
                       "timing": "10 back-to-back launches between CUDA events"}}


def bench_c1(args, world, dev):
    """BASELINE.json configs[0] on the GPU: one 1237x822 view's importance map and LAS on 100k
    SH3 Gaussians (all masked). Latency-bound at this size, so each is timed both through the
    public call and as a CUDA-graph replay of the same launches ("use CUDA
    graphs for C1"); the reference times are one process on the host."""
    import torch

    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200.synth import random_cloud_torch, synth_views_torch
    view = synth_views_torch(1, H, W, seed=3000, device=dev)
    out = torch.empty((1, H, W), dtype=torch.float64, device=dev)
    n = 100_000
    pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=7, device=dev)
    scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
    mask = torch.ones(n, dtype=torch.bool, device=dev)
    c = igs.SplitConstants()

    def events(fn, k=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        b.record()
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b) / k, world)

    def graphed(fn):
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(2):
                fn()
        torch.cuda.current_stream(dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return events(g.replay)

    res = {"config": {"workload": "BASELINE.json configs[0]: 1 x 1237x822 RGB f64 view; LAS on "
                                  "100k SH3 Gaussians, all masked",
                      "timing": "20 calls / graph replays between CUDA events"}}
    edge = lambda: igs.importance_batch(view, out=out)  # noqa: E731
    res["edge_public_ms"] = round(events(edge), 4)
    split = lambda: igs.las_split.split_async(scene, mask, c)  # noqa: E731
    try:
        res["edge_graph_ms"] = round(graphed(edge), 4)
        res["las_graph_ms"] = round(graphed(split), 4)   # pre-pass + guarded apply, no read
    except RuntimeError as e:  # capture unsupported here: keep the public-call numbers
        res["graph_error"] = str(e)[:160]
    pristine = {k: getattr(scene, k)[:n].clone() for k in ("_pos", "_ls", "_op")}
    times = []
    for it in range(23):
        for k, v in pristine.items():
            getattr(scene, k)[:n].copy_(v)
        scene._set_count(n)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        igs.las_split_batch(scene, mask, c)
        b.record()
        torch.cuda.synchronize()
        if it >= 3:
            times.append(a.elapsed_time(b))
    res["las_public_ms"] = round(max_over_ranks(statistics.median(times), world), 4)
    res["edge_MPix_s"] = round(PX / (min(res.get("edge_graph_ms", 1e9), res["edge_public_ms"])
                                     * 1e-3) / 1e6, 1)
    res["las_Gaussians_s"] = round(n / (min(res.get("las_graph_ms", 1e9), res["las_public_ms"])
                                        * 1e-3), 1)
    if world == 1 and not args.no_cpu and ref_kind() == "reference":
        from paper_2603_08661_b200.synth import synth_view
        fn = ref_edge_fn()
        v = synth_view(H, W, 3000)
        fn(v)
        t0 = time.perf_counter()
        fn(v)
        res["cpu_reference_edge_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
        rate, _, _ = cpu_las_rate(n)
        res["cpu_reference_las_ms"] = round(n / rate * 1e3, 1)
    return res


def bench_las(args, world, dev, peak, peak_src):
    import torch

    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200 import _lib
    from paper_2603_08661_b200.synth import random_cloud_torch, random_stats

    n = LAS_N
    pos, ls, q, o, sh = random_cloud_torch(n, 16, seed=101, device=dev)
    scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n, device=dev)
    pristine = {k: getattr(scene, k).clone() for k in ("_pos", "_ls", "_op")}
    mask = torch.ones(n, dtype=torch.bool, device=dev)

    def restore():
        for k, v in pristine.items():
            getattr(scene, k)[:n].copy_(v[:n])
        scene._set_count(n)

    # all-masked LAS through the public call: las_split_batch = fused pre-pass + device-guarded
    # apply, then the 16-byte summary read
    times = []
    steps = max(3, min(args.steps, 20))
    for it in range(args.warmup + steps):
        restore()
        torch.cuda.synchronize()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        igs.las_split_batch(scene, mask)
        c.record()
        torch.cuda.synchronize()
        if it >= args.warmup:
            times.append(a.elapsed_time(c))
    ms = max_over_ranks(statistics.median(times), world)
    # the apply kernel alone: K back-to-back launches on one prepared workspace between two
    # events (each launch moves the same bytes; the scene is restored afterwards), so the
    # per-launch time excludes the host's launch gap that the public-call timing above sees
    restore()
    prep = igs.las_split.prepare(scene, mask, igs.SplitConstants())
    ns, fl = (int(v) for v in prep.summary.cpu())
    L = _lib.lib()
    alpha, log_alpha, log_gamma, beta = igs.SplitConstants().device_constants()
    apply_args = (scene._pos.data_ptr(), scene._ls.data_ptr(), scene._rot.data_ptr(),
                  scene._op.data_ptr(), scene._sh.data_ptr(), scene._sh.shape[1] * 3, n, 2 * n,
                  prep.mask_u8.data_ptr(), alpha, log_alpha, log_gamma, beta, 0,
                  prep.ws.data_ptr(), prep.ws.numel(), _lib.stream_handle(dev))
    K = 10
    for _ in range(2):
        _lib.check(L.igs_las_apply(*apply_args), "las bench")
    torch.cuda.synchronize()
    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        L.igs_las_apply(*apply_args)
    c.record()
    torch.cuda.synchronize()
    ms_kernel = max_over_ranks(a.elapsed_time(c) / K, world)
    # the public call's device work: igs_las_split (cooperative pre-pass + guarded apply), K
    # back-to-back launches at the same count (each splits all n parents again)
    summ = torch.zeros(2, dtype=torch.int64, device=dev)
    split_args = apply_args[:13] + (prep.ws.data_ptr(), prep.ws.numel(), summ.data_ptr(),
                                    _lib.stream_handle(dev))
    restore()
    for _ in range(2):
        _lib.check(L.igs_las_split(*split_args), "las bench")
    torch.cuda.synchronize()
    a.record()
    for _ in range(K):
        L.igs_las_split(*split_args)
    c.record()
    torch.cuda.synchronize()
    ms_split = max_over_ranks(a.elapsed_time(c) / K, world)
    restore()
    achieved = n * LAS_BYTES_PER_SPLIT / (ms_kernel * 1e-3) / 1e9
    # full densify_step on the same cloud: select (take = 5% = 50k) + LAS
    grad, edge = random_stats(n, seed=7)
    dsteps = []
    for it in range(args.warmup + steps):
        restore()
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
        if it >= args.warmup:
            dsteps.append(a.elapsed_time(c))
    ds_ms = max_over_ranks(statistics.median(dsteps), world)
    las_traffic = ncu_traffic().get("las_apply_kernel_bytes_per_split")
    res = {"metric": "LAS Gaussians/s", "value": round(world * n / (ms * 1e-3), 1),
           "unit": "Gaussians/s", "ms_per_step": round(ms, 4),
           "config": {"workload": "las_split_batch, 1M Gaussians all masked, SH degree 3 "
                                  "(59 fp32/Gaussian), capacity 2M (BASELINE.json configs[2])",
                      "l2": "500 MB moved per step >> L2"},
           "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(achieved / peak, 4),
                        "traffic": (round(las_traffic * n) if las_traffic else None),
                        "kernel": "las_apply_kernel", "algorithmic_bytes_per_split": 500,
                        "kernel_ms": round(ms_kernel, 4), "peak_source": peak_src,
                        "split_device_ms": round(ms_split, 4),
                        "split_device_frac": round(n * LAS_BYTES_PER_SPLIT / (ms_split * 1e-3)
                                                   / 1e9 / peak, 4),
                        "timing": "kernel_ms: 10 back-to-back apply launches between CUDA "
                                  "events; split_device_ms: 10 back-to-back igs_las_split "
                                  "(cooperative pre-pass + guarded apply); ms_per_step: the "
                                  "public las_split_batch call, CUDA events around it (host work, "
                                  "the launches, the spin on the pinned pre-pass summary; the "
                                  "apply pass ends before the closing event)"},
           "densify_step": {"ms": round(ds_ms, 4), "n": n, "split": ev.split,
                            "eligible": ev.eligible,
                            "note": "select (radix top-k, take=ceil(0.05 N)) + LAS + the "
                                    "statistics reset, public densify_step(); the host reads "
                                    "the pinned select count and split summary"}}
    if world == 1 and not args.no_cpu:
        rate, kind, sample = cpu_las_rate()
        res["cpu_baseline"] = {"value": round(rate, 1), "unit": "Gaussians/s", "cores": 1,
                               "kind": kind, "sample": sample}
    return res


DENSIFY_N = 6_000_000
UHD_VIEWS = 128


def bench_scene_io(args, dev, n=6_000_000):
    """.igsp load / save of a 6M-Gaussian colour-only cloud (BASELINE.json configs[3] size,
    14 floats per record = 336 MB) between a page-cached file and device columns: pinned
    read + per-column H2D + GPU quaternion renormalisation, and D2H + atomic rename. Host
    wall clock around synchronised calls (the path is host IO)."""
    import shutil
    import tempfile

    import numpy as np
    import torch

    import paper_2603_08661_b200 as igs
    rng = np.random.default_rng(11)
    q = rng.normal(size=(n, 4)).astype(np.float32)
    sc = igs.Scene3(rng.normal(size=(n, 3)).astype(np.float32),
                    rng.uniform(-1, 1, (n, 3)).astype(np.float32), q,
                    rng.normal(size=n).astype(np.float32), rng.random((n, 3)).astype(np.float32),
                    capacity=n, device=dev)
    d = tempfile.mkdtemp(prefix="igsp_bench_")
    try:
        path = os.path.join(d, "cloud.igsp")
        igs.write_scene(sc, path)
        nbytes = os.path.getsize(path)
        reps = 3
        for _ in range(1):
            igs.read_scene(path, capacity=n + n // 20, device=dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            back = igs.read_scene(path, capacity=n + n // 20, device=dev)
        torch.cuda.synchronize()
        rd = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            igs.write_scene(back, path)
        wr = (time.perf_counter() - t0) / reps
        res = {"metric": "scene file GB/s", "gaussians": n, "bytes": nbytes,
               "read_GBps": round(nbytes / rd / 1e9, 2), "read_ms": round(rd * 1e3, 2),
               "write_GBps": round(nbytes / wr / 1e9, 2), "write_ms": round(wr * 1e3, 2),
               "config": {"workload": "read_scene / write_scene, 6M Gaussians, colour-only "
                                      "records (io_cli.py:83-134), page-cached file in /tmp",
                          "timing": "host wall clock, 3 reps after 1 warm-up"}}
        if ref_kind() == "reference" and not args.no_cpu:
            if REF_PATH not in sys.path:
                sys.path.insert(0, REF_PATH)
            from splitkit.io_cli import read_scene as ref_read
            ref_read(path)
            t0 = time.perf_counter()
            ref_read(path)
            res["cpu_baseline"] = {"read_GBps": round(nbytes / (time.perf_counter() - t0) / 1e9, 2),
                                   "cores": 1, "kind": "reference",
                                   "sample": "one splitkit.io_cli.read_scene of the same file"}
        return res
    finally:
        shutil.rmtree(d, ignore_errors=True)


def bench_uhd(args, world, dev, peak):
    """BASELINE.json configs[4]: 3840x2160 views, 128 per GPU (1024 over 8 GPUs); the same
    fused launch as the headline, weak scaling, max-over-ranks device time."""
    import torch

    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200.synth import UHD_H, UHD_W, synth_views_torch
    views = synth_views_torch(UHD_VIEWS, UHD_H, UHD_W, seed=5000, device=dev, distinct=4)
    out = torch.empty((UHD_VIEWS, UHD_H, UHD_W), dtype=torch.float64, device=dev)
    for _ in range(2):
        igs.importance_batch(views, out=out)
    steps = max(2, min(args.steps, 5))
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        igs.importance_batch(views, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps, world)
    px = UHD_VIEWS * UHD_H * UHD_W
    achieved = px * BYTES_PER_PX_F64 / (ms * 1e-3) / 1e9
    del views, out
    torch.cuda.empty_cache()
    return {"metric": "edge-map MPix/s", "value": round(world * px / (ms * 1e-3) / 1e6, 3),
            "unit": "MPix/s", "ms_per_step": round(ms, 3), "steps": steps, "scaling": "weak",
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4)},
            "config": {"workload": f"{UHD_VIEWS} x 3840x2160 RGB f64 views per GPU "
                                   "(BASELINE.json configs[4]: 1024 over 8 GPUs)",
                       "l2": "25 GB of input per GPU >> L2"}}


def bench_densify_sharded(args, world, rank, dev):
    """BASELINE.json configs[3]: the full densify step on a 6M-Gaussian SH3 cloud split in
    contiguous shards over the ranks (strong scaling: 6M total at every N).  One step =
    keys + one 256 KB histogram all-reduce + boundary records all-gather + finalize + the
    guarded split of each shard + one host read of the plan; max over ranks of the median
    step."""
    import torch

    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200 import sharded
    from paper_2603_08661_b200.synth import random_cloud_torch, random_stats

    lo, hi = sharded.shard_range(DENSIFY_N, rank, world)
    k = hi - lo
    pos, ls, q, o, sh = random_cloud_torch(k, 16, seed=301 + rank, device=dev)
    scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * k, device=dev)
    pristine = {name: getattr(scene, name)[:k].clone() for name in ("_pos", "_ls", "_op")}
    grad, edge = random_stats(k, seed=17 + rank)
    grad_t = torch.from_numpy(grad).to(dev)
    comm = sharded.Comm()
    caps = sharded.global_counts(scene, comm)
    cfg = igs.DensifyConfig(budget=2 * DENSIFY_N)
    times, ev = [], None
    steps = max(3, min(args.steps, 20))
    for it in range(args.warmup + steps):
        for name, v in pristine.items():
            getattr(scene, name)[:k].copy_(v)
        scene._set_count(k)
        sharded.detach(scene)   # the restored cloud is again a contiguous shard
        sharded.attach(scene, comm, caps)
        stats = igs.DensifyStats(k, device=dev)
        stats._grad_sum.copy_(grad_t)
        stats._accum_count = 1
        stats.set_edge_score(edge)
        torch.cuda.synchronize()
        barrier(world)
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ev = sharded.densify_step_sharded(scene, stats, cfg, 2000, comm, caps=caps)
        c.record()
        torch.cuda.synchronize()
        if it >= args.warmup:
            times.append(a.elapsed_time(c))
    ms = max_over_ranks(statistics.median(times), world)
    algo = DENSIFY_N * 17 + ev.split * 500  # select bytes + LAS bytes
    return {"metric": "densify step Gaussians/s", "value": round(DENSIFY_N / (ms * 1e-3), 1),
            "unit": "Gaussians/s", "ms_per_step": round(ms, 4), "scaling": "strong",
            "n_gpus": world, "split": ev.split, "eligible": ev.eligible,
            "count_after": ev.count_after,
            "algorithmic_GBps_per_gpu": round(algo / world / (ms * 1e-3) / 1e9, 1),
            "config": {"workload": "densify_step_sharded on a 6M-Gaussian SH3 cloud, contiguous "
                                   f"shards of {k} per GPU, take = ceil(0.05 N) = 300k "
                                   "(BASELINE.json configs[3])",
                       "collectives": "1 x 256 KB all-reduce + 1 all-gather of 64 KB "
                                      "boundary records per rank per step "
                                      + ("(NCCL)" if world > 1 else "(none at N=1)")}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-las", action="store_true")
    ap.add_argument("--no-uhd", action="store_true")
    ap.add_argument("--no-check", action="store_true",
                    help="skip the oracle check of a sample of the timed views")
    args = ap.parse_args()
    args.steps_given = args.steps is not None
    if args.steps is None:
        args.steps = 50
    args.warmup = max(args.warmup, 0)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, world, int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup()
    try:
        run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
