"""Seeded synthetic workloads: Mip-NeRF360-shaped views,
random Gaussian clouds with SH degree 3, and densification statistics.

Everything is generated with numpy on the host (the same arrays feed the CUDA
path and the CPU oracle); ``*_torch`` helpers build the same data directly on a
CUDA device for the large benchmark configurations.
"""

from __future__ import annotations

import numpy as np

VIEW_H, VIEW_W = 822, 1237        # Mip-NeRF360 images_4 shape (1237 x 822)
UHD_H, UHD_W = 2160, 3840


def synth_view(h=VIEW_H, w=VIEW_W, seed=1000, dtype=np.float64):
    """8-bit-quantised smooth RGB view in [0, 1]: sin/cos carrier per channel + N(0, .05)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    out = np.empty((h, w, 3))
    for c in range(3):
        ph = rng.uniform(0, 2 * np.pi)
        out[..., c] = 0.5 + 0.5 * np.sin(xx / 37 + ph) * np.cos(yy / 53 - ph)
    out += rng.normal(0, 0.05, out.shape)
    return (np.floor(np.clip(out, 0, 1) * 255 + 0.5) / 255).astype(dtype)


def synth_views(b, h=VIEW_H, w=VIEW_W, seed0=1000, dtype=np.float64):
    return np.stack([synth_view(h, w, seed0 + v, dtype) for v in range(b)])


def synth_views_torch(b, h=VIEW_H, w=VIEW_W, seed=1000, device="cuda", dtype=None,
                      distinct=8):
    """(b, h, w, 3) float64 views on `device`: `distinct` host-generated views tiled
    over the batch with a per-view roll so no two views are byte-identical."""
    import torch
    dtype = dtype or torch.float64
    base = torch.from_numpy(synth_views(min(distinct, b), h, w, seed)).to(device, dtype)
    out = torch.empty((b, h, w, 3), dtype=dtype, device=device)
    for v in range(b):
        out[v] = torch.roll(base[v % base.shape[0]], shifts=(7 * (v // base.shape[0]),), dims=(1,))
    return out


def random_cloud(n, sh_coeffs=16, seed=101):
    """Random Gaussians after test_acceptance.py:50-58 (+ SH block (n, K, 3))."""
    rng = np.random.default_rng(seed)
    pos = rng.normal(0.0, 1.0, (n, 3)).astype(np.float32)
    ls = rng.uniform(-0.7, 0.7, (n, 3)).astype(np.float32)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    o = rng.normal(0.0, 1.5, n).astype(np.float32)
    sh = np.empty((n, sh_coeffs, 3), dtype=np.float32)
    sh[:, 0, :] = rng.random((n, 3))
    if sh_coeffs > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.1, (n, sh_coeffs - 1, 3))
    return pos, ls, q.astype(np.float32), o, sh


def random_cloud_torch(n, sh_coeffs=16, seed=101, device="cuda"):
    """Same distributions as random_cloud, generated on the device (large N)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f = dict(device=device, dtype=torch.float32)
    pos = torch.randn((n, 3), generator=g, **f)
    ls = torch.rand((n, 3), generator=g, **f) * 1.4 - 0.7
    q = torch.randn((n, 4), generator=g, device=device, dtype=torch.float64)
    q = (q / q.norm(dim=1, keepdim=True)).float()
    o = torch.randn((n,), generator=g, **f) * 1.5
    sh = torch.randn((n, sh_coeffs, 3), generator=g, **f) * 0.1
    sh[:, 0, :] = torch.rand((n, 3), generator=g, **f)
    return pos, ls, q, o, sh


def random_stats(n, seed=7):
    """grad_norm ~ Exp(mean 2e-4), edge_score ~ U(0,1), float64."""
    rng = np.random.default_rng(seed)
    return rng.exponential(2e-4, n), rng.random(n)
