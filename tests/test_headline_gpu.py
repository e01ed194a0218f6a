"""Parity at the benchmark's own batch sizes.

The fused edge kernel keeps a ring of RING = 16 survivor-list / candidate slots (csrc/edge.cu);
a batch of more than 16 views reuses slot v % 16 for view v once view v - 16 has retired.
These tests run the shapes the bench times (BASELINE.json configs[1]: 200 x 1237x822; configs[4]:
3840x2160 views; configs[3]: a 6M-Gaussian sharded select) and compare with the oracle
(oracle/edge.py restates edge_pipeline.py:42-135 bit for bit; oracle/select.py restates
densify_controller.py:80-106).
"""

import numpy as np
import pytest
import torch

from oracle import edge as OE
from oracle import select as OS

pytestmark = pytest.mark.gpu

H, W = 822, 1237


def _mixed_views(n):
    """n full-size views: seeded synthetic photos plus structured classes (flat 16-px blocks,
    a white rectangle, uniform noise, a constant image) spread through the batch."""
    from paper_2603_08661_b200.synth import synth_view
    rng = np.random.default_rng(21)
    views = np.empty((n, H, W, 3))
    for v in range(n):
        kind = v % 12
        if kind == 5:
            views[v] = np.kron(rng.integers(0, 256, (52, 78, 3)), np.ones((16, 16, 1)))[:H, :W] / 255
        elif kind == 8:
            views[v] = 0.0
            views[v, 100 + v:500, 200:900 - v] = 1.0
        elif kind == 11:
            views[v] = rng.random((H, W, 3))
        elif v == 13:
            views[v] = 0.25   # no positive survivors: the median is 1.0 and no apply work
        else:
            views[v] = synth_view(H, W, 4000 + v)
    return views


def test_ring_wraps_48_views_bit_exact_three_repeats():
    """48 full-size views (the ring wraps twice), three launches in a row, every pixel."""
    import paper_2603_08661_b200 as b
    views = _mixed_views(48)
    want = [OE.importance_pipeline(views[v]) for v in range(views.shape[0])]
    dev_views = torch.from_numpy(views).cuda()
    out = torch.empty((views.shape[0], H, W), dtype=torch.float64, device="cuda")
    for rep in range(3):
        out.fill_(-1.0)
        b.importance_batch(dev_views, out=out)
        got = out.cpu().numpy()
        bad = [v for v in range(len(want)) if not np.array_equal(got[v], want[v])]
        assert not bad, f"repeat {rep}: views {bad} differ from the oracle"


def test_bench_batch_200_views_sample_bit_exact():
    """The bench's exact workload (synth_views_torch(200), one launch): sampled views on both
    sides of every ring wrap, against the oracle on the same device-generated views."""
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200.synth import synth_views_torch
    views = synth_views_torch(200, H, W, seed=1000, device="cuda")
    out = torch.empty((200, H, W), dtype=torch.float64, device="cuda")
    for _ in range(2):
        b.importance_batch(views, out=out)
    torch.cuda.synchronize()
    for v in (0, 15, 16, 17, 31, 32, 63, 100, 143, 184, 199):
        want = OE.importance_pipeline(views[v].cpu().numpy())
        assert np.array_equal(out[v].cpu().numpy(), want), f"view {v}"


def test_uhd_two_views_bit_exact():
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200.synth import UHD_H, UHD_W, synth_view
    views = np.stack([synth_view(UHD_H, UHD_W, 5000), synth_view(UHD_H, UHD_W, 5001)])
    got = b.importance_batch(views)
    for v in range(2):
        assert np.array_equal(got[v], OE.importance_pipeline(views[v])), f"UHD view {v}"


def test_uhd_ring_wrap_sample_bit_exact():
    """20 UHD views in one launch (ring wraps), sampled against the oracle."""
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200.synth import UHD_H, UHD_W, synth_views_torch
    views = synth_views_torch(20, UHD_H, UHD_W, seed=5000, device="cuda", distinct=4)
    out = b.importance_batch(views)
    for v in (0, 16, 19):
        want = OE.importance_pipeline(views[v].cpu().numpy())
        assert np.array_equal(out[v].cpu().numpy(), want), f"UHD view {v}"


def test_sharded_select_6M_world1_equals_single_and_oracle():
    """configs[3]'s cloud size through the sharded protocol at world 1."""
    import paper_2603_08661_b200 as b
    from paper_2603_08661_b200 import sharded
    n = 6_000_000
    rng = np.random.default_rng(66)
    grad, edge = rng.exponential(2e-4, n), np.round(rng.random(n), 3)   # many exact ties
    for step in (2000, 500):
        cfg = b.DensifyConfig(budget=2 * n)
        st = b.DensifyStats(n)
        st._grad_sum.copy_(torch.from_numpy(grad))
        st._accum_count = 1
        st.set_edge_score(edge)
        single = b.select_candidates(st, cfg, step, n).cpu().numpy()
        got = sharded.select_candidates_sharded(st, cfg, step, n, n).cpu().numpy()
        warm = OS.is_warmup_step(500, 15000, 500, 3, step)
        want, _ = OS.select_candidates(grad, edge, warm, "product", 2e-4, 0.05, n)
        assert int(want.sum()) == 300_000
        np.testing.assert_array_equal(single, want)
        np.testing.assert_array_equal(got, want)
