"""The reference trainer's use of the densification API (splat2d.py:382-398), through the drop-in.

Every iteration the trainer re-assigns each scene column from the host, folds np.hypot of the
positional gradients into the running statistics, and at densify steps assigns
``stats.edge_score = sample_scores(importance, scene.positions)`` and calls ``densify_step``.
Here the same sequence runs on a GPU ``Scene2`` and, in parallel, on the oracle (numpy dict
scene + oracle/select.py + oracle/las.py); events and columns must agree at every densify step.
"""

import numpy as np
import pytest
import torch

from oracle import edge as OE
from oracle import las as OL
from oracle import select as OS

pytestmark = pytest.mark.gpu


def test_trainer_assignment_idiom_matches_oracle():
    import paper_2603_08661_b200 as igs
    from paper_2603_08661_b200.synth import synth_view
    h, w, n0, cap = 96, 128, 48, 160
    target = synth_view(h, w, 77)
    imp = igs.importance_pipeline(target)
    assert np.array_equal(imp, OE.importance_pipeline(target))
    rng = np.random.default_rng(5)
    f32 = np.float32
    ref = {"positions": np.stack([rng.uniform(0, w - 1, n0), rng.uniform(0, h - 1, n0)], 1).astype(f32),
           "log_scales": np.full((n0, 2), np.log(w / 16.0), f32),
           "thetas": rng.uniform(-1, 1, n0).astype(f32),
           "opacity_logits": rng.normal(0, 1, n0).astype(f32),
           "colors": rng.random((n0, 3)).astype(f32), "capacity": cap}
    scene = igs.Scene2(ref["positions"], ref["log_scales"], ref["thetas"], ref["opacity_logits"],
                       ref["colors"], capacity=cap)
    cfg = igs.DensifyConfig(budget=cap, interval=4, window_start=4, window_end=40,
                            grad_threshold=0.05)
    stats = igs.DensifyStats(scene.count)
    gsum, accum = np.zeros(n0), 0
    events = 0
    for step in range(41):
        n = scene.count
        g = rng.normal(0, 0.1, (n, 2))
        lr = 0.5
        # splat2d.py:382-391: every column re-assigned from host arrays
        ref["positions"] = (ref["positions"].astype(np.float64) - lr * g).astype(f32)
        ref["log_scales"] = (ref["log_scales"].astype(np.float64) - 0.01 * g).astype(f32)
        ref["thetas"] = (ref["thetas"].astype(np.float64) - 0.01 * g[:, 0]).astype(f32)
        ref["opacity_logits"] = (ref["opacity_logits"].astype(np.float64) + 0.01 * g[:, 1]).astype(f32)
        ref["colors"] = np.clip(ref["colors"].astype(np.float64) - 0.01 * g[:, :1], 0, 1).astype(f32)
        for col in ("positions", "log_scales", "thetas", "opacity_logits", "colors"):
            setattr(scene, col, ref[col])
        # splat2d.py:393-394
        norms = np.hypot(g[:, 0], g[:, 1])
        igs.accumulate_grads(stats, norms)
        gsum, accum = gsum + norms, accum + 1
        if not igs.is_densify_step(cfg, step):
            continue
        # splat2d.py:396-398
        stats.edge_score = igs.sample_scores(imp, scene.positions)
        edge = OE.sample_scores(imp, ref["positions"].astype(np.float64))
        assert np.array_equal(stats.edge_score.cpu().numpy(), edge)
        ev = igs.densify_step(scene, stats, cfg, step)
        warm = igs.is_warmup_step(cfg, step)
        headroom = cap - n
        mask, elig = OS.select_candidates(OS.grad_norm(gsum, accum), edge, warm, cfg.policy,
                                          cfg.grad_threshold, cfg.growth_cap, headroom)
        ref = OL.las_split_batch_2d(ref, mask)
        assert (ev.eligible, ev.split, ev.count_after) == (elig, int(mask.sum()),
                                                           len(ref["positions"])), step
        got = scene.to_numpy()
        for col in ("log_scales", "thetas", "colors"):
            assert np.array_equal(got[col], ref[col]), (step, col)
        np.testing.assert_allclose(got["positions"], ref["positions"], rtol=1e-5, atol=1e-4)
        np.testing.assert_allclose(got["opacity_logits"], ref["opacity_logits"], rtol=1e-5,
                                   atol=1e-5)
        # continue from the device values (the float32 exp/cos of the split may differ in the
        # last place from numpy's SIMD loops; SURVEY.md 8(c) tolerance)
        ref = dict(got)
        ref.pop("capacity")
        ref["capacity"] = cap
        gsum, accum = np.zeros(scene.count), 0
        events += ev.split > 0
    assert events >= 3 and scene.count > n0
