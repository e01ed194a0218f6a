"""Parity of the CUDA selection (radix top-k) and densify_step with the oracle / golden vectors."""

import numpy as np
import pytest
import torch
from numpy.testing import assert_array_equal

from conftest import load_golden
from oracle import select as OS

pytestmark = pytest.mark.gpu

SEL = load_golden("select")


def B():
    import paper_2603_08661_b200 as b
    return b


def gpu_stats(grad_sum, accum, edge):
    b = B()
    st = b.DensifyStats(len(grad_sum))
    st._grad_sum.copy_(torch.from_numpy(np.asarray(grad_sum, np.float64)))
    st._accum_count = int(accum)
    st.set_edge_score(edge)
    return st


def test_golden_selection_bit_exact():
    b = B()
    for name, c in sorted(SEL.items()):
        if not name.startswith("s"):
            continue
        step, cap, headroom, thr = c["params"]
        cfg = b.DensifyConfig(budget=10 * len(c["edge"]), growth_cap=float(cap),
                              policy=str(c["policy"]), grad_threshold=float(thr))
        st = gpu_stats(c["grad_sum"], c["accum"], c["edge"])
        mask = b.select_candidates(st, cfg, int(step), int(headroom))
        assert_array_equal(mask.cpu().numpy(), c["mask"], err_msg=name)


@pytest.mark.parametrize("n", [1, 7, 1000, 65_537, 1_000_000])
@pytest.mark.parametrize("tied", [False, True])
def test_large_random_vs_oracle(n, tied):
    b = B()
    rng = np.random.default_rng(n + tied)
    grad = rng.exponential(2e-4, n)
    edge = rng.random(n)
    if tied:
        grad = np.round(grad, 4)
        edge = np.round(edge, 1)
    for step, policy, cap in ((2000, "product", 0.05), (500, "product", 0.3),
                              (2000, "grad", 0.5), (2000, "edge", 1.0)):
        cfg = b.DensifyConfig(budget=10 * n, growth_cap=cap, policy=policy)
        st = gpu_stats(grad * 3, 3, edge)
        headroom = n
        got = b.select_candidates(st, cfg, step, headroom).cpu().numpy()
        warm = OS.is_warmup_step(500, 15000, 500, 3, step)
        want, _ = OS.select_candidates(OS.grad_norm(grad * 3, 3), edge, warm, policy,
                                       cfg.grad_threshold, cap, headroom)
        assert_array_equal(got, want, err_msg=f"{step} {policy} {cap}")


def test_order_semantics_nan_inf_signed_zero():
    b = B()
    edge = np.array([0.5, np.nan, -0.0, 0.0, 0.5, np.inf, 0.25])
    st = gpu_stats(np.ones(7), 1, edge)
    cfg = b.DensifyConfig(budget=100, growth_cap=1.0)
    for headroom, want in ((1, [5]), (3, [0, 4, 5]), (5, [0, 2, 4, 5, 6]),
                           (6, [0, 2, 3, 4, 5, 6]), (7, list(range(7)))):
        m = b.select_candidates(st, cfg, 500, headroom).cpu().numpy()
        assert_array_equal(np.flatnonzero(m), want, err_msg=str(headroom))


def test_reference_known_answers():
    b = B()
    cfg = lambda **k: b.DensifyConfig(budget=1000, **k)
    st = gpu_stats([1.0] * 4, 1, [0.5] * 4)
    m = b.select_candidates(st, cfg(grad_threshold=0.5, growth_cap=0.5), 2000, 2)
    assert_array_equal(m.cpu().numpy(), [True, True, False, False])
    st = gpu_stats(np.ones(60), 1, np.ones(60))
    assert int(b.select_candidates(st, cfg(grad_threshold=0.5), 2000, 60).sum()) == 3
    st = gpu_stats(np.ones(40), 1, np.ones(40))
    assert int(b.select_candidates(st, cfg(grad_threshold=0.5, growth_cap=1.0), 2000,
                                   3).sum()) == 3
    with pytest.raises(ValueError):
        b.select_candidates(st, cfg(), 2000, -1)
    st = gpu_stats([0.0, 0.0, 0.0], 1, [0.9, 0.1, 0.5])
    assert_array_equal(b.select_candidates(st, cfg(), 500, 1).cpu().numpy(), [1, 0, 0])


def test_golden_densify_step():
    b = B()
    for name, c in sorted(SEL.items()):
        if not name.startswith("d"):
            continue
        colors = c["in_colors"]
        s = b.Scene3(c["in_positions"], c["in_log_scales"], c["in_rotations"],
                     c["in_opacity_logits"], colors, 260)
        st = gpu_stats(c["grad_sum"], 1, c["edge"])
        ev = b.densify_step(s, st, b.DensifyConfig(budget=260, growth_cap=0.2), int(c["step"]))
        assert [ev.step, ev.eligible, ev.split, ev.count_after] == list(c["event"]), name
        got = s.to_numpy()
        assert_array_equal(got["rotations"], c["out_rotations"])
        assert_array_equal(got["log_scales"], c["out_log_scales"])
        assert_array_equal(got["colors"], c["out_colors"])
        np.testing.assert_allclose(got["positions"], c["out_positions"], rtol=0, atol=1e-5)
        assert len(st) == s.count


def test_densify_step_guards():
    b = B()
    z = np.zeros((4, 3), np.float32)
    q = np.tile(np.array([1, 0, 0, 0], np.float32), (4, 1))
    s = b.Scene3(z, z, q, np.zeros(4, np.float32), np.ones((4, 3), np.float32), 4)
    with pytest.raises(ValueError):
        b.densify_step(s, b.DensifyStats(4), b.DensifyConfig(budget=4), 123)
    with pytest.raises(ValueError):
        b.densify_step(s, b.DensifyStats(3), b.DensifyConfig(budget=4), 500)
    st = b.DensifyStats(4)
    b.accumulate_grads(st, np.ones(4))
    ev = b.densify_step(s, st, b.DensifyConfig(budget=4, grad_threshold=0.0, growth_cap=1.0), 2000)
    assert ev.split == 0 and s.count == 4 and ev.eligible == 4


def test_accumulate_position_grads_matches_numpy_hypot():
    """splat2d.py:393-394: accumulate_grads(stats, np.hypot(g[:, 0], g[:, 1])), fused."""
    b = B()
    rng = np.random.default_rng(31)
    n = 100_003
    st = b.DensifyStats(n)
    want = np.zeros(n)
    for it, dt in enumerate((np.float64, np.float32, np.float64)):
        g = (rng.standard_normal((n, 2)) * np.exp(rng.uniform(-30, 5, (n, 1)))).astype(dt)
        g[:5] = [[0.0, 0.0], [-0.0, 3.0], [np.inf, 1.0], [1e-310, 1e-310], [3e300, 4e300]]
        b.accumulate_position_grads(st, g)
        with np.errstate(all="ignore"):
            want = want + np.hypot(g[:, 0], g[:, 1]).astype(np.float64)
        assert st._accum_count == it + 1
    np.testing.assert_array_equal(st._grad_sum.cpu().numpy(), want)
    with pytest.raises(ValueError):
        b.accumulate_position_grads(st, np.zeros((n, 3)))


def test_hypot_bit_exact_wide_range():
    """The device glibc hypot (shared by the edge kernel's survivor magnitudes) against np.hypot
    on 4M pairs: every exponent range, axis-aligned zeros, signed zeros, subnormals, inf/NaN."""
    b = B()
    rng = np.random.default_rng(77)
    n = 1 << 22
    with np.errstate(over="ignore"):
        g = rng.standard_normal((n, 2)) * np.exp2(rng.integers(-1074, 1023, (n, 2)).clip(-1070, 1000))
        g[::7, 1] = 0.0
        g[::11, 0] = -0.0
        g[::13] = g[::13] * np.exp2(rng.integers(-60, 60, (len(g[::13]), 1)))  # near-equal and far
        g[1::17, 1] = g[1::17, 0] * rng.uniform(0.999, 1.001, len(g[1::17]))
    sp = np.array([[np.inf, 1.0], [np.nan, np.inf], [np.nan, 1.0], [5e-324, 0.0], [0.0, 0.0],
                   [1.7976931348623157e308, 1.7976931348623157e308], [3.0, 4.0], [1e-300, 1e-310]])
    g[:len(sp)] = sp
    st = b.DensifyStats(n)
    b.accumulate_position_grads(st, g)
    with np.errstate(all="ignore"):
        want = 0.0 + np.hypot(g[:, 0], g[:, 1])
    got = st._grad_sum.cpu().numpy()
    np.testing.assert_array_equal(got.view(np.int64)[~np.isnan(want)],
                                  want.view(np.int64)[~np.isnan(want)])
    assert np.isnan(got[np.isnan(want)]).all()


def test_stats_reset_is_lazy_and_exact():
    """DensifyStats.reset writes nothing: pending rows read as zeros, the first position-gradient
    accumulation stores 0.0 + h (IGS_ACCUM_STORE), an edge-score assignment overwrites, and the
    selection sees the same values as after an explicit zero fill (densify_controller.py:23-63)."""
    b = B()
    rng = np.random.default_rng(5)
    n = 50_001
    st = b.DensifyStats(n)
    g1 = rng.standard_normal((n, 2))
    b.accumulate_position_grads(st, g1)
    st._buf.fill_(np.nan)            # stale contents must never leak through a reset
    st.reset(n + 7)
    assert len(st) == n + 7
    assert torch.equal(st.grad_norm, torch.zeros(n + 7, dtype=torch.float64, device="cuda"))
    st._buf.fill_(np.nan)
    g2 = (rng.standard_normal((n + 7, 2)) * 3).astype(np.float32)
    g2[0] = [-0.0, -0.0]
    b.accumulate_position_grads(st, g2)
    b.accumulate_position_grads(st, g2.astype(np.float64))
    with np.errstate(all="ignore"):
        want = (0.0 + np.hypot(g2[:, 0], g2[:, 1]).astype(np.float64)) + np.hypot(
            g2[:, 0].astype(np.float64), g2[:, 1].astype(np.float64))
    got = st._grad_sum.cpu().numpy()
    np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))
    assert torch.equal(st.edge_score, torch.zeros(n + 7, dtype=torch.float64, device="cuda"))
    st.reset()
    st._buf.fill_(np.nan)
    e = rng.uniform(0, 1, n + 7)
    st.edge_score = e
    assert torch.equal(st.edge_score.cpu(), torch.from_numpy(e))
    assert torch.equal(st._grad_sum, torch.zeros(n + 7, dtype=torch.float64, device="cuda"))
    st.reset()
    st._buf.fill_(np.nan)
    b.accumulate_grads(st, np.ones(n + 7))
    assert torch.equal(st._grad_sum.cpu(), torch.ones(n + 7, dtype=torch.float64))
