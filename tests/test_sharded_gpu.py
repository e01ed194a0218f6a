"""GPU parity of the sharded densification path (igs_shard_* + the guarded split on shards).

* world 1 (no process group): the sharded radix select through the real CUDA kernels equals
  the single-launch select and the oracle, bit for bit;
* world 2 over gloo, both ranks on cuda:0 (the box has one GPU; NCCL refuses two ranks per
  device): densify_step_sharded + gather_scene reproduce the single-device densify_step
  exactly (masks, counts, every column in the reference's global layout)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT
from oracle import select as OS

pytestmark = pytest.mark.gpu


def _stats(b, grad_sum, accum, edge, device="cuda"):
    st = b.DensifyStats(len(grad_sum), device=device)
    st._grad_sum.copy_(torch.from_numpy(np.asarray(grad_sum, np.float64)))
    st._accum_count = int(accum)
    st.set_edge_score(edge)
    return st


@pytest.mark.parametrize("n", [1, 5, 3000, 65_536 * 3 + 7, 750_000])
@pytest.mark.parametrize("tied", [False, True])
def test_world1_sharded_select_equals_single(n, tied):
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200 import sharded
    rng = np.random.default_rng(n * 2 + tied)
    grad, edge = rng.exponential(2e-4, n), rng.random(n)
    if tied:
        grad, edge = np.round(grad, 4), np.round(edge, 1)
    for step, policy, cap in ((2000, "product", 0.05), (500, "edge", 0.3), (2000, "grad", 1.0)):
        cfg = b.DensifyConfig(budget=10 * n, growth_cap=cap, policy=policy)
        st = _stats(b, grad * 3, 3, edge)
        got = sharded.select_candidates_sharded(st, cfg, step, n, n).cpu().numpy()
        single = b.select_candidates(st, cfg, step, n).cpu().numpy()
        warm = OS.is_warmup_step(500, 15000, 500, 3, step)
        want, _ = OS.select_candidates(OS.grad_norm(grad * 3, 3), edge, warm, policy, 2e-4, cap, n)
        np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(single, want)


@pytest.mark.parametrize("n,world_cap", [(20_000, None), (3_000, 8)])
def test_world1_degenerate_boundary_bucket(n, world_cap):
    """Every score equal (a warm-up event with all edge scores 0): the whole eligible set is
    one boundary bucket -- larger than the kernel's selection capacity (device-sort path), or
    than a small record (re-run path); ties break by index as the stable argsort does."""
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200 import sharded
    grad, edge = np.full(n, 3e-4), np.zeros(n)
    for step in (500, 2000):
        cfg = b.DensifyConfig(budget=10 * n, growth_cap=0.3)
        st = _stats(b, grad, 1, edge)
        got = sharded.select_candidates_sharded(st, cfg, step, n, n,
                                                record_cap=world_cap).cpu().numpy()
        warm = OS.is_warmup_step(500, 15000, 500, 3, step)
        want, _ = OS.select_candidates(grad, edge, warm, "product", 2e-4, 0.3, n)
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("policy,step", [("edge", 500), ("product", 2000)])
def test_world1_special_scores_large(policy, step):
    """NaN, signed zeros, negatives, subnormals, huge and infinite scores scattered through a
    large array (the keys' digits come from their high words, with the low word only for the
    NaN key and the subnormal corner): bit-exact with the oracle at several take sizes."""
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200 import sharded
    n = 100_003
    rng = np.random.default_rng(77)
    edge = rng.random(n)
    special = np.array([np.nan, -0.0, 0.0, -1.5, 5e-324, 1e-310, -1e-310, 2.2e-308, 1e300,
                        np.inf, -np.inf, 3e-19, 4.0, 7.9])
    pick = rng.choice(n, n // 50, replace=False)
    edge[pick] = special[rng.integers(0, len(special), len(pick))]
    grad = rng.exponential(3e-4, n)
    for cap in (0.001, 0.05, 0.5):
        cfg = b.DensifyConfig(budget=10 * n, growth_cap=cap, policy=policy)
        st = _stats(b, grad, 1, edge)
        got = sharded.select_candidates_sharded(st, cfg, step, n, n).cpu().numpy()
        warm = OS.is_warmup_step(500, 15000, 500, 3, step)
        want, _ = OS.select_candidates(grad, edge, warm, policy, 2e-4, cap, n)
        np.testing.assert_array_equal(got, want, err_msg=f"{policy} cap={cap}")


def test_world1_order_semantics():
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200 import sharded
    edge = np.array([0.5, np.nan, -0.0, 0.0, 0.5, np.inf, 0.25])
    cfg = b.DensifyConfig(budget=100, growth_cap=1.0, policy="edge")
    for take in range(1, 8):
        st = _stats(b, np.ones(7), 1, edge)
        got = sharded.select_candidates_sharded(st, cfg, 500, take, 7).cpu().numpy()
        want, _ = OS.select_candidates(np.ones(7), edge, True, "edge", 2e-4, 1.0, take)
        np.testing.assert_array_equal(got, want)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cloud(n, seed):
    from paper_2603_08661_b200.synth import random_cloud
    return random_cloud(n, 16, seed=seed)


def _worker(rank, world, port, n, q, backend="gloo"):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0) if backend == "nccl" else None)
    try:
        import paper_2603_08661_b200 as b
        from paper_2603_08661_b200 import sharded
        pos, ls, qq, o, sh = _cloud(n, 11)
        rng = np.random.default_rng(12)
        grad, edge = rng.exponential(3e-4, n), np.round(rng.random(n), 2)
        lo, hi = sharded.shard_range(n, rank, world)
        k = hi - lo
        scene = b.Scene3(pos[lo:hi], ls[lo:hi], qq[lo:hi], o[lo:hi], sh[lo:hi], capacity=2 * k)
        st = _stats(b, grad[lo:hi], 1, edge[lo:hi])
        cfg = b.DensifyConfig(budget=2 * n, growth_cap=0.3)
        ev = sharded.densify_step_sharded(scene, st, cfg, 2000)
        full = sharded.gather_scene(scene, k)
        q.put((rank, (ev.step, ev.eligible, ev.split, ev.count_after),
               {kk: v.cpu().numpy() for kk, v in full.items()}))
    finally:
        dist.destroy_process_group()


def _worker_events(rank, world, port, n, q, skew):
    """Two consecutive densify events on the shards (the second one's ties break by the
    global indices the first one gave the children); `skew`: every high score on rank 0,
    whose own rows are too few to hold its children -- the global capacity still does."""
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_08661_b200 as b
        from paper_2603_08661_b200 import sharded
        pos, ls, qq, o, sh, grads, edges = _event_inputs(n, skew)
        lo, hi = sharded.shard_range(n, rank, world)
        k = hi - lo
        cap = k + (n // 8 if skew else k)   # the shards' reservations differ from the global one
        scene = b.Scene3(pos[lo:hi], ls[lo:hi], qq[lo:hi], o[lo:hi], sh[lo:hi], capacity=cap)
        caps = sharded.global_counts(scene, sharded.Comm())
        glob_cap = 3 * n
        caps = [(c, glob_cap // world + (glob_cap % world if r == 0 else 0))
                for r, (c, _) in enumerate(caps)]
        cfg = b.DensifyConfig(budget=glob_cap, growth_cap=0.3)
        evs = []
        for step, (grad, edge) in zip((2000, 2500), zip(grads, edges)):
            gi = scene._gidx[:scene.count].cpu().numpy() if hasattr(scene, "_gidx") else \
                np.arange(lo, hi)
            st = _stats(b, grad[gi], 1, edge[gi])
            ev = sharded.densify_step_sharded(scene, st, cfg, step, caps=caps)
            evs.append((ev.step, ev.eligible, ev.split, ev.count_after))
            if step == 2000:   # the children follow the reference's numbering after event 1
                full1 = sharded.gather_scene(scene)
                q.put(("event1", rank, {kk: v.cpu().numpy() for kk, v in full1.items()}))
                sharded.reshard(scene)
        full = sharded.gather_scene(scene)
        q.put((rank, evs, {kk: v.cpu().numpy() for kk, v in full.items()}))
    finally:
        dist.destroy_process_group()


def _event_inputs(n, skew):
    pos, ls, qq, o, sh = _cloud(n, 21)
    rng = np.random.default_rng(22)
    total = n + int(np.ceil(0.3 * n)) + 10
    grads = [rng.exponential(3e-4, total), rng.exponential(3e-4, total)]
    edges = [np.round(rng.random(total), 1), np.round(rng.random(total), 1)]  # many ties
    if skew:
        for e in edges:
            e[: n // 2] += 2.0     # the first half of the global array (rank 0) wins
    return pos, ls, qq, o, sh, grads, edges


@pytest.mark.parametrize("skew", [False, True])
def test_sharded_two_events_match_single_device(skew):
    import paper_2603_08661_b200 as b
    n, world = 9_001, 2
    pos, ls, qq, o, sh, grads, edges = _event_inputs(n, skew)
    scene = b.Scene3(pos, ls, qq, o, sh, capacity=3 * n)
    cfg = b.DensifyConfig(budget=3 * n, growth_cap=0.3)
    want_ev, want1 = [], None
    for step, (grad, edge) in zip((2000, 2500), zip(grads, edges)):
        st = _stats(b, grad[:scene.count], 1, edge[:scene.count])
        ev = b.densify_step(scene, st, cfg, step)
        want_ev.append((ev.step, ev.eligible, ev.split, ev.count_after))
        if want1 is None:
            want1 = scene.to_numpy()
    want = scene.to_numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_events, args=(r, world, port, n, q, skew))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2 * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for item in res:
        if item[0] == "event1":
            _, rank, full = item
            ref = want1
        else:
            rank, evs, full = item
            assert evs == want_ev, rank
            ref = want
        for col in ("positions", "log_scales", "rotations", "opacity_logits", "sh"):
            np.testing.assert_array_equal(full[col], ref[col], err_msg=f"{col} rank {rank}")


@pytest.mark.parametrize("world,backend", [(2, "gloo"), (1, "nccl")])
def test_sharded_densify_step_matches_single_device(world, backend):
    """world 2 over gloo (two ranks on the one GPU), and world 1 over NCCL (the production
    backend's collectives on device buffers)."""
    import paper_2603_08661_b200 as b
    n = 20_001
    pos, ls, qq, o, sh = _cloud(n, 11)
    rng = np.random.default_rng(12)
    grad, edge = rng.exponential(3e-4, n), np.round(rng.random(n), 2)
    scene = b.Scene3(pos, ls, qq, o, sh, capacity=2 * n)
    st = _stats(b, grad, 1, edge)
    cfg = b.DensifyConfig(budget=2 * n, growth_cap=0.3)
    ev = b.densify_step(scene, st, cfg, 2000)
    want = scene.to_numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, backend))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, evt, full in res:
        assert evt == (ev.step, ev.eligible, ev.split, ev.count_after), rank
        for col in ("positions", "log_scales", "rotations", "opacity_logits", "sh"):
            np.testing.assert_array_equal(full[col], want[col], err_msg=f"{col} rank {rank}")


def test_world1_sharded_select_reference_golden():
    """The sharded radix select against the reference's own masks (tests/golden/select.npz),
    including the non-finite statistics cases (NaN / inf scores and gradient sums)."""
    import paper_2603_08661_b200 as b
    from conftest import load_golden
    from paper_2603_08661_b200 import sharded
    for name, c in load_golden("select").items():
        if not name.startswith("s"):
            continue
        step, cap, headroom, thr = c["params"]
        n = len(c["grad_sum"])
        cfg = b.DensifyConfig(budget=10 * n, growth_cap=float(cap), policy=str(c["policy"]),
                              grad_threshold=float(thr))
        st = _stats(b, c["grad_sum"], int(c["accum"]), c["edge"])
        got = sharded.select_candidates_sharded(st, cfg, int(step), int(headroom), n)
        np.testing.assert_array_equal(got.cpu().numpy(), c["mask"], err_msg=name)


@pytest.mark.parametrize("k_sh", [1, 4, 9, 16])
def test_world1_sharded_step_sh_sizes(k_sh):
    """The list-mode guarded split of the sharded step for every SH row width (3, 12, 27 and
    48 floats: scalar, float4 and the unrolled clone paths) against the single-device step."""
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200 import sharded
    n = 5_003
    pos, ls, qq, o, sh = _cloud(n, 31)
    sh = np.ascontiguousarray(np.repeat(sh[:, :1, :], k_sh, axis=1) +
                              np.arange(k_sh, dtype=np.float32)[None, :, None])
    rng = np.random.default_rng(32)
    grad, edge = rng.exponential(3e-4, n), rng.random(n)
    want = b.Scene3(pos, ls, qq, o, sh, capacity=2 * n)
    ev_w = b.densify_step(want, _stats(b, grad, 1, edge), b.DensifyConfig(budget=2 * n,
                                                                          growth_cap=0.2), 2000)
    got = b.Scene3(pos, ls, qq, o, sh, capacity=2 * n)
    ev_g = sharded.densify_step_sharded(got, _stats(b, grad, 1, edge),
                                        b.DensifyConfig(budget=2 * n, growth_cap=0.2), 2000)
    assert (ev_g.eligible, ev_g.split, ev_g.count_after) == \
        (ev_w.eligible, ev_w.split, ev_w.count_after)
    gw, gg = want.to_numpy(), got.to_numpy()
    for col in ("positions", "log_scales", "rotations", "opacity_logits", "sh"):
        np.testing.assert_array_equal(gg[col], gw[col], err_msg=col)


def test_world1_sharded_step_2d_scene():
    """A 2-D scene through the sharded step (flags without quaternions, the guarded 2-D split)
    against the single-device densify_step."""
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200 import sharded
    n = 4_001
    rng = np.random.default_rng(41)
    cols = (rng.normal(0, 5, (n, 2)), rng.uniform(-1, 1, (n, 2)), rng.uniform(-3, 3, n),
            rng.normal(0, 1.5, n), rng.random((n, 3)))
    grad, edge = rng.exponential(3e-4, n), rng.random(n)
    want = b.Scene2(*cols, capacity=2 * n)
    ev_w = b.densify_step(want, _stats(b, grad, 1, edge), b.DensifyConfig(budget=2 * n,
                                                                          growth_cap=0.2), 2000)
    got = b.Scene2(*cols, capacity=2 * n)
    ev_g = sharded.densify_step_sharded(got, _stats(b, grad, 1, edge),
                                        b.DensifyConfig(budget=2 * n, growth_cap=0.2), 2000)
    assert (ev_g.eligible, ev_g.split, ev_g.count_after) == \
        (ev_w.eligible, ev_w.split, ev_w.count_after)
    gw, gg = want.to_numpy(), got.to_numpy()
    for col in ("positions", "log_scales", "thetas", "opacity_logits", "colors"):
        np.testing.assert_array_equal(gg[col], gw[col], err_msg=col)
