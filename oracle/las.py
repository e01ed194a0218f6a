"""Oracle: Long-Axis-Split restated on the CPU in float32 numpy (TEST INFRASTRUCTURE ONLY).

Restates ``splitkit.las_split.las_split_batch`` and the helpers it calls
(``/root/reference/pkg/src/splitkit/las_split.py:52-179``,
``core.py:17-58,151-157``) operation by operation in float32, the dtype the
reference stores scenes in.  The one extension over the reference is the
spherical-harmonics block: the reference ``Scene3`` carries ``colors`` (N, 3),
the SH degree-0 case; here a scene carries ``sh`` (N, K, 3) whose K
coefficient triplets are cloned to the appended child exactly like
``colors`` is at ``las_split.py:177`` (``colors == sh[:, 0, :]``).

Scenes are plain dicts of numpy arrays with keys ``positions`` (N,3),
``log_scales`` (N,3), ``rotations`` (N,4), ``opacity_logits`` (N,),
``sh`` (N,K,3) and ``capacity`` (int).
"""

from __future__ import annotations

import math

import numpy as np


class BudgetError(RuntimeError):
    """las_split.py:26-27."""


def sigmoid(x):
    """core.py:17-21."""
    x = np.asarray(x)
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-x))


def logit(p):
    """core.py:24-29 (ValueError unless 0 < p < 1 everywhere)."""
    p = np.asarray(p)
    if not np.all((p > 0.0) & (p < 1.0)):
        raise ValueError("logit requires all values strictly inside (0, 1)")
    return np.log(p / (1.0 - p))


def quat_to_rotmat(q):
    """core.py:32-58: row-major R from (w, x, y, z).

    Batch-global rule (core.py:45-46): ALL rows are renormalised iff ANY row's
    norm strays more than 1e-4 from 1; zero / non-finite norms raise.
    """
    q = np.asarray(q)
    norm = np.sqrt((q * q).sum(axis=-1))
    if not np.all(np.isfinite(norm)) or np.any(norm == 0.0):
        raise ValueError("zero or non-finite quaternion")
    if np.any(np.abs(norm - 1.0) > 1e-4):
        q = q / norm[..., None]
    w, x, y, z = (q[..., i] for i in range(4))
    r = np.empty(q.shape[:-1] + (3, 3), dtype=q.dtype)
    r[..., 0, 0] = 1.0 - 2.0 * (y * y + z * z)
    r[..., 0, 1] = 2.0 * (x * y - w * z)
    r[..., 0, 2] = 2.0 * (x * z + w * y)
    r[..., 1, 0] = 2.0 * (x * y + w * z)
    r[..., 1, 1] = 1.0 - 2.0 * (x * x + z * z)
    r[..., 1, 2] = 2.0 * (y * z - w * x)
    r[..., 2, 0] = 2.0 * (x * z - w * y)
    r[..., 2, 1] = 2.0 * (y * z + w * x)
    r[..., 2, 2] = 1.0 - 2.0 * (x * x + y * y)
    return r


def check_constants(alpha=0.5, gamma_axis=0.85, beta=0.6):
    """SplitConstants validation, las_split.py:43-49."""
    if not 0.0 < alpha < 1.0:
        raise ValueError("alpha must be in (0, 1)")
    if not 0.0 < gamma_axis <= 1.0:
        raise ValueError("gamma_axis must be in (0, 1]")
    if not 0.0 < beta <= 1.0:
        raise ValueError("beta must be in (0, 1]")


def split_columns(positions, log_scales, rotations, opacity_logits,
                  alpha=0.5, gamma_axis=0.85, beta=0.6):
    """_split_common + _split3_columns (las_split.py:78-106) in the storage dtype."""
    dt = log_scales.dtype.type
    log_alpha, log_gamma = dt(math.log(alpha)), dt(math.log(gamma_axis))
    rows = np.arange(len(log_scales))
    l_idx = np.argmax(log_scales, axis=-1)          # first maximum wins
    long_ls = log_scales[rows, l_idx]
    offset = np.exp(long_ls) * dt(alpha)
    child_ls = log_scales + log_gamma
    child_ls[rows, l_idx] = long_ls + log_alpha
    child_o = logit(sigmoid(opacity_logits) * dt(beta)).astype(log_scales.dtype, copy=False)
    rot = quat_to_rotmat(rotations).reshape(-1, 9)
    column = np.take_along_axis(rot, l_idx[:, None] + np.array([0, 3, 6]), axis=-1)
    disp = column * offset[:, None]
    return positions + disp, positions - disp, child_ls, child_o


def las_split_batch(scene, mask, alpha=0.5, gamma_axis=0.85, beta=0.6):
    """las_split.py:158-179 on a dict scene; returns a NEW dict (inputs untouched).

    Parents keep their slot and receive the +offset child; -offset children
    are appended in ascending parent order (rank = prefix count of the mask).
    """
    check_constants(alpha, gamma_axis, beta)
    n = len(scene["positions"])
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != (n,):
        raise ValueError(f"mask length {mask.shape} does not match scene count {n}")
    k = int(mask.sum())
    if n + k > scene["capacity"]:
        raise BudgetError(f"splitting {k} of {n} primitives exceeds capacity {scene['capacity']}")
    out = {key: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v)
           for key, v in scene.items()}
    if k == 0:
        return out
    idx = np.flatnonzero(mask)
    pa, pb, cls, co = split_columns(scene["positions"][idx], scene["log_scales"][idx],
                                    scene["rotations"][idx], scene["opacity_logits"][idx],
                                    alpha, gamma_axis, beta)
    out["positions"][idx] = pa
    out["log_scales"][idx] = cls
    out["opacity_logits"][idx] = co
    out["positions"] = np.concatenate([out["positions"], pb])
    out["log_scales"] = np.concatenate([out["log_scales"], cls])
    out["rotations"] = np.concatenate([out["rotations"], scene["rotations"][idx]])
    out["opacity_logits"] = np.concatenate([out["opacity_logits"], co])
    out["sh"] = np.concatenate([out["sh"], scene["sh"][idx]])
    return out


def split_columns_2d(positions, log_scales, thetas, opacity_logits,
                     alpha=0.5, gamma_axis=0.85, beta=0.6):
    """_split_common + _split2_columns (las_split.py:78-99, 109-117): the long-axis column of
    the 2-D rotation [[cos, -sin], [sin, cos]] -- (cos, sin) for axis 0, (-sin, cos) for 1."""
    dt = log_scales.dtype.type
    log_alpha, log_gamma = dt(math.log(alpha)), dt(math.log(gamma_axis))
    rows = np.arange(len(log_scales))
    l_idx = np.argmax(log_scales, axis=-1)
    long_ls = log_scales[rows, l_idx]
    offset = np.exp(long_ls) * dt(alpha)
    child_ls = log_scales + log_gamma
    child_ls[rows, l_idx] = long_ls + log_alpha
    child_o = logit(sigmoid(opacity_logits) * dt(beta)).astype(log_scales.dtype, copy=False)
    c, s = np.cos(thetas), np.sin(thetas)
    column = np.where((l_idx == 0)[:, None], np.stack([c, s], -1), np.stack([-s, c], -1))
    disp = column * offset[:, None]
    return positions + disp, positions - disp, child_ls, child_o


def las_split_batch_2d(scene, mask, alpha=0.5, gamma_axis=0.85, beta=0.6):
    """las_split.py:182-197 on a dict scene (positions (N,2), log_scales (N,2), thetas (N,),
    opacity_logits (N,), colors (N,3), capacity); returns a NEW dict."""
    check_constants(alpha, gamma_axis, beta)
    n = len(scene["positions"])
    mask = np.asarray(mask, dtype=bool)
    if mask.shape != (n,):
        raise ValueError(f"mask length {mask.shape} does not match scene count {n}")
    k = int(mask.sum())
    if n + k > scene["capacity"]:
        raise BudgetError(f"splitting {k} of {n} primitives exceeds capacity {scene['capacity']}")
    out = {key: (np.array(v, copy=True) if isinstance(v, np.ndarray) else v)
           for key, v in scene.items()}
    if k == 0:
        return out
    idx = np.flatnonzero(mask)
    pa, pb, cls, co = split_columns_2d(scene["positions"][idx], scene["log_scales"][idx],
                                       scene["thetas"][idx], scene["opacity_logits"][idx],
                                       alpha, gamma_axis, beta)
    out["positions"][idx] = pa
    out["log_scales"][idx] = cls
    out["opacity_logits"][idx] = co
    out["positions"] = np.concatenate([out["positions"], pb])
    out["log_scales"] = np.concatenate([out["log_scales"], cls])
    out["thetas"] = np.concatenate([out["thetas"], scene["thetas"][idx]])
    out["opacity_logits"] = np.concatenate([out["opacity_logits"], co])
    out["colors"] = np.concatenate([out["colors"], scene["colors"][idx]])
    return out
