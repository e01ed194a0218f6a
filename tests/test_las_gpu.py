"""Parity of the CUDA Long-Axis-Split with the oracle and the reference's golden vectors."""

import math

import numpy as np
import pytest
import torch
from numpy.testing import assert_array_equal

from conftest import load_golden
from oracle import las as OL

pytestmark = pytest.mark.gpu

LAS = load_golden("las")


def B():
    import paper_2603_08661_b200 as b
    return b


def assert_las_close(got, want, label=""):
    """rotations, SH and child log-scales bit-exact; positions within
    1e-5 (|p| + |disp|); opacity within 1e-5 max(1, |o|)."""
    for col in ("rotations", "log_scales", "sh"):
        assert_array_equal(got[col], want[col], err_msg=f"{label} {col}")
    gp, wp = got["positions"].astype(np.float64), want["positions"].astype(np.float64)
    assert gp.shape == wp.shape, label
    with np.errstate(all="ignore"):
        scale = np.abs(wp) + np.exp(want["log_scales"].astype(np.float64)).max(axis=1,
                                                                               keepdims=True) * 2
        close = np.abs(gp - wp) <= 1e-5 * scale
    # non-finite results (NaN / inf log-scales or positions) must match exactly
    nonfin = ~np.isfinite(wp)
    close[nonfin] = (gp[nonfin] == wp[nonfin]) | (np.isnan(gp[nonfin]) & np.isnan(wp[nonfin]))
    assert close.all(), f"{label} positions"
    go, wo = got["opacity_logits"].astype(np.float64), want["opacity_logits"].astype(np.float64)
    assert (np.abs(go - wo) <= 1e-5 * np.maximum(1.0, np.abs(wo))).all(), f"{label} opacity"


def scene_dict(c, prefix):
    return {"positions": c[f"{prefix}_positions"], "log_scales": c[f"{prefix}_log_scales"],
            "rotations": c[f"{prefix}_rotations"], "opacity_logits": c[f"{prefix}_opacity_logits"],
            "sh": c[f"{prefix}_colors"][:, None, :], "capacity": int(c["capacity"])}


def gpu_scene(d):
    return B().Scene3(d["positions"], d["log_scales"], d["rotations"], d["opacity_logits"],
                      d["sh"], d["capacity"])


@pytest.mark.parametrize("case", sorted(LAS))
def test_golden_las(case):
    b = B()
    c = LAS[case]
    consts = b.SplitConstants(*c["constants"]) if "constants" in c else b.SplitConstants()
    s = gpu_scene(scene_dict(c, "in"))
    b.las_split_batch(s, c["mask"], consts)
    assert s.count == len(c["out_positions"])
    assert_las_close(s.to_numpy(), scene_dict(c, "out"), case)


def test_sh_degree3_clone_vs_oracle():
    b = B()
    from paper_2603_08661_b200.synth import random_cloud
    n = 20_000
    pos, ls, q, o, sh = random_cloud(n, 16, seed=5)
    rng = np.random.default_rng(6)
    for p in (0.05, 0.5, 1.0):
        mask = rng.random(n) < p
        d = {"positions": pos, "log_scales": ls, "rotations": q, "opacity_logits": o, "sh": sh,
             "capacity": 2 * n + 3}
        want = OL.las_split_batch(d, mask)
        s = gpu_scene(d)
        b.las_split_batch(s, torch.from_numpy(mask).cuda())
        assert_las_close(s.to_numpy(), want, f"p={p}")


@pytest.mark.parametrize("sh_coeffs", [1, 16])
def test_sparse_list_mode_vs_oracle(sh_coeffs):
    """igs_las_split_sparse (the list-mode apply densify_step uses) gives the tile-mode results
    for every mask density, and leaves the scene untouched on a capacity overflow."""
    b = B()
    from paper_2603_08661_b200 import las_split as LS
    from paper_2603_08661_b200.synth import random_cloud
    n = 50_000
    pos, ls, q, o, sh = random_cloud(n, sh_coeffs, seed=17 + sh_coeffs)
    rng = np.random.default_rng(sh_coeffs)
    for p in (0.0, 0.001, 0.05, 0.5, 1.0):
        mask = rng.random(n) < p
        d = {"positions": pos, "log_scales": ls, "rotations": q, "opacity_logits": o, "sh": sh,
             "capacity": 2 * n}
        want = OL.las_split_batch(d, mask)
        s = gpu_scene(d)
        summ = LS.split_async(s, torch.from_numpy(mask).cuda(), b.SplitConstants(), sparse=True)
        n_split, flags = (int(v) for v in summ.cpu())
        assert n_split == int(mask.sum()) and flags == 0
        LS.finish_split(s, n_split, flags)
        assert_las_close(s.to_numpy(), want, f"p={p}")
    d = {"positions": pos, "log_scales": ls, "rotations": q, "opacity_logits": o, "sh": sh,
         "capacity": n + 10}
    s = gpu_scene(d)
    before = s.to_numpy()
    mask = np.zeros(n, bool)
    mask[::1000] = True                              # 50 splits > 10 free rows
    summ = LS.split_async(s, torch.from_numpy(mask).cuda(), b.SplitConstants(), sparse=True)
    with pytest.raises(b.BudgetError):
        LS.finish_split(s, *(int(v) for v in summ.cpu()))
    after = s.to_numpy()
    assert s.count == n
    for col in before:
        assert_array_equal(after[col], before[col], err_msg=col)


def test_million_all_masked_acceptance_ratios():
    """Acceptance criterion 1 (test_acceptance.py:61-104) on 1M splits, plus oracle parity."""
    b = B()
    from paper_2603_08661_b200.synth import random_cloud
    n = 1_000_000
    pos, ls, q, o, sh = random_cloud(n, 16, seed=101)
    d = {"positions": pos, "log_scales": ls, "rotations": q, "opacity_logits": o, "sh": sh,
         "capacity": 2 * n}
    s = gpu_scene(d)
    b.las_split_batch(s, np.ones(n, bool))
    got = s.to_numpy()
    assert s.count == 2 * n
    want = OL.las_split_batch(d, np.ones(n, bool))
    assert_las_close(got, want, "1M")
    first, second = slice(0, n), slice(n, 2 * n)
    P = got["positions"].astype(np.float64)
    mid = (P[first] + P[second]) / 2
    assert np.abs(mid - pos).max() <= 1e-6 * 4   # float32 positions of magnitude ~4
    ratios = np.exp(got["log_scales"][first].astype(np.float64) - ls.astype(np.float64))
    la = np.argmax(ls, axis=1)
    rows = np.arange(n)
    assert np.abs(ratios[rows, la] / 0.5 - 1).max() <= 1e-6
    other = np.ones((n, 3), bool)
    other[rows, la] = False
    assert np.abs(ratios[other] / 0.85 - 1).max() <= 1e-6
    sig = lambda x: 1 / (1 + np.exp(-x.astype(np.float64)))
    assert np.abs(sig(got["opacity_logits"][first]) / sig(o) - 0.6).max() <= 1e-6


def test_errors_leave_scene_untouched():
    b = B()
    z = np.zeros((4, 3), np.float32)
    q = np.tile(np.array([1, 0, 0, 0], np.float32), (4, 1))
    s = b.Scene3(z, z, q, np.zeros(4, np.float32), np.ones((4, 3), np.float32), 5)
    with pytest.raises(b.BudgetError):
        b.las_split_batch(s, np.ones(4, bool))
    with pytest.raises(ValueError):
        b.las_split_batch(s, np.ones(3, bool))
    s2 = b.Scene3(z, z, q, np.zeros(4, np.float32), np.ones((4, 3), np.float32), 8)
    s2._rot[2] = 0.0
    before = s2.to_numpy()
    with pytest.raises(ValueError):
        b.las_split_batch(s2, np.ones(4, bool))
    after = s2.to_numpy()
    assert s2.count == 4
    for k in ("positions", "log_scales", "opacity_logits"):
        assert_array_equal(after[k], before[k])
    # logit domain: sigmoid(-100) underflows to 0 in float32 -> ValueError (core.py:27-28)
    s3 = b.Scene3(z, z, q, np.array([0, -100, 0, 0], np.float32), np.ones((4, 3), np.float32), 8)
    with pytest.raises(ValueError):
        b.las_split_batch(s3, np.array([False, True, False, False]))
    assert s3.count == 4
    # the same parent unmasked is fine
    b.las_split_batch(s3, np.array([True, False, False, False]))
    assert s3.count == 5


def test_empty_mask_and_worked_example():
    b = B()
    s = b.Scene3(np.zeros((1, 3)), np.zeros((1, 3)), [[1, 0, 0, 0]], [0.0], [[1, 1, 1]], 4)
    b.las_split_batch(s, [False])
    assert s.count == 1
    b.las_split_batch(s, [True])
    g = s.to_numpy()
    np.testing.assert_allclose(g["positions"], [[0.5, 0, 0], [-0.5, 0, 0]], atol=1e-7)
    np.testing.assert_allclose(g["log_scales"][0], [math.log(.5), math.log(.85), math.log(.85)],
                               atol=1e-6)
    np.testing.assert_allclose(g["opacity_logits"], -0.847298, atol=1e-6)


def test_batch_equals_sequential_random_scenes():
    """Acceptance criterion 3 (batch == sequential) via the oracle, 200 random scenes."""
    b = B()
    rng = np.random.default_rng(103)
    for _ in range(200):
        n = int(rng.integers(1, 300))
        d = {"positions": rng.normal(0, 1, (n, 3)).astype(np.float32),
             "log_scales": rng.uniform(-.7, .7, (n, 3)).astype(np.float32),
             "rotations": (lambda q: (q / np.linalg.norm(q, axis=1, keepdims=True)))(
                 rng.normal(size=(n, 4))).astype(np.float32),
             "opacity_logits": rng.normal(0, 1.5, n).astype(np.float32),
             "sh": rng.random((n, 1, 3)).astype(np.float32), "capacity": 2 * n + 1}
        mask = rng.random(n) < 0.4
        s = gpu_scene(d)
        b.las_split_batch(s, mask)
        assert_las_close(s.to_numpy(), OL.las_split_batch(d, mask))


LAS2D = load_golden("las2d")


@pytest.mark.parametrize("case", sorted(LAS2D))
def test_golden_las2d(case):
    """las_split_batch_2d: log-scales, thetas, colours bit-exact; positions / opacities within
    the north-star tolerance (numpy's float32 exp / log / sin / cos are not correctly rounded)."""
    b = B()
    c = LAS2D[case]
    sc = b.Scene2(c["in_positions"], c["in_log_scales"], c["in_thetas"], c["in_opacity_logits"],
                  c["in_colors"], capacity=int(c["capacity"]))
    a, g, be = (float(x) for x in c["constants"])
    b.las_split_batch_2d(sc, c["mask"], b.SplitConstants(alpha=a, gamma_axis=g, beta=be))
    got = sc.to_numpy()
    for k in ("log_scales", "thetas", "colors"):
        assert_array_equal(got[k], c[f"out_{k}"], err_msg=k)
    want_p, p_in = c["out_positions"], c["in_positions"]
    n = len(p_in)
    scale = np.abs(want_p).copy()
    scale[:n] += np.abs(want_p[:n] - p_in)
    assert (np.abs(got["positions"] - want_p) <= 1e-5 * (scale + 1e-30) + 1e-7).all()
    wo = c["out_opacity_logits"]
    assert (np.abs(got["opacity_logits"] - wo) <= 1e-5 * np.maximum(1.0, np.abs(wo))).all()


def test_las2d_errors():
    b = B()
    sc = b.Scene2(np.zeros((4, 2)), np.zeros((4, 2)), np.zeros(4), np.zeros(4), np.zeros((4, 3)),
                  capacity=5)
    with pytest.raises(b.BudgetError):
        b.las_split_batch_2d(sc, np.ones(4, bool))
    with pytest.raises(ValueError):
        b.las_split_batch_2d(sc, np.ones(3, bool))
    assert sc.count == 4
    b.las_split_batch_2d(sc, np.zeros(4, bool))
    assert sc.count == 4


def test_densify_step_scene2_matches_oracle():
    """densify_step on a 2-D scene (densify_controller.py:125-147 dispatches to
    las_split_batch_2d): the fused select + guarded 2-D split against the oracle."""
    from oracle import select as OS
    b = B()
    rng = np.random.default_rng(8)
    n = 5000
    cols = {"positions": rng.normal(size=(n, 2)), "log_scales": rng.uniform(-0.7, 0.7, (n, 2)),
            "thetas": rng.uniform(-np.pi, np.pi, n), "opacity_logits": rng.normal(0, 1.5, n),
            "colors": rng.random((n, 3))}
    cols = {k: v.astype(np.float32) for k, v in cols.items()}
    sc = b.Scene2(cols["positions"], cols["log_scales"], cols["thetas"], cols["opacity_logits"],
                  cols["colors"], capacity=n + 600)
    grad, edge = rng.exponential(3e-4, n), rng.random(n)
    st = b.DensifyStats(n)
    b.accumulate_grads(st, grad)
    st.set_edge_score(edge)
    cfg = b.DensifyConfig(budget=n + 600)
    ev = b.densify_step(sc, st, cfg, 2000)
    mask, elig = OS.select_candidates(grad, edge, False, "product", cfg.grad_threshold,
                                      cfg.growth_cap, 600)
    assert (ev.eligible, ev.split, ev.count_after) == (elig, int(mask.sum()), n + int(mask.sum()))
    k = cfg.split_constants
    want = OL.las_split_batch_2d(dict(cols, capacity=n + 600), mask, k.alpha, k.gamma_axis, k.beta)
    got = sc.to_numpy()
    for c in ("log_scales", "thetas", "colors"):
        assert_array_equal(got[c], want[c], err_msg=c)
    wp = want["positions"].astype(np.float64)
    assert (np.abs(got["positions"] - wp) <= 1e-5 * (np.abs(wp) + 1.0)).all()
    wo = want["opacity_logits"]
    assert (np.abs(got["opacity_logits"] - wo) <= 1e-5 * np.maximum(1.0, np.abs(wo))).all()
    assert len(st) == sc.count


def test_fused_split_leaves_scene_untouched_on_errors():
    """igs_las_split decides on the device: BudgetError and the logit-domain ValueError leave
    every column as it was (las_split.py:158-179 raise before mutating)."""
    b = B()
    n = 64
    q = np.tile([1.0, 0, 0, 0], (n, 1))
    sc = b.Scene3(np.arange(3 * n).reshape(n, 3), np.zeros((n, 3)), q, np.zeros(n),
                  np.ones((n, 3)), capacity=n + 10)
    before = sc.to_numpy()
    with pytest.raises(b.BudgetError):
        b.las_split_batch(sc, np.ones(n, bool))
    sc2 = b.Scene3(np.arange(3 * n).reshape(n, 3), np.zeros((n, 3)), q, np.full(n, 1e9),
                   np.ones((n, 3)), capacity=2 * n)
    before2 = sc2.to_numpy()
    with pytest.raises(ValueError):
        b.las_split_batch(sc2, np.ones(n, bool), b.SplitConstants(beta=1.0))
    for s_, bf in ((sc, before), (sc2, before2)):
        after = s_.to_numpy()
        assert s_.count == n
        for col in ("positions", "log_scales", "rotations", "opacity_logits", "sh"):
            assert_array_equal(after[col], bf[col])
