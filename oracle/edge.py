"""Oracle: edge-importance pipeline restated on the CPU (TEST INFRASTRUCTURE ONLY).

Restates ``splitkit.edge_pipeline`` (``/root/reference/pkg/src/splitkit/
edge_pipeline.py``) in float64 numpy, spelling out the arithmetic order of the
third-party kernels the reference delegates to, so the CUDA path can be held
to bit-exact parity:

* ``scipy.ndimage.convolve/correlate(mode="nearest")`` -- scipy's C routine
  ``NI_Correlate`` (scipy 1.18.1; reference pins ``scipy>=1.10``) keeps the
  taps with ``|w| > DBL_EPSILON``, starts every output at ``0.0`` and adds
  ``x * w`` for the kept taps in C (row-major) order of the weight array, one
  rounded multiply and one rounded add per tap (no FMA).  Out-of-image reads
  replicate the nearest edge pixel.
* ``np.hypot`` -- glibc >= 2.35 ``__hypot`` (non-FMA x86-64 build): scaled
  Borges correction of ``sqrt(ax*ax + ay*ay)``; restated in
  :func:`hypot_glibc` and pinned against ``np.hypot`` in the tests.
* ``np.arctan2``/``np.mod`` -- libm ``atan2`` then numpy's float remainder.
* ``np.median`` -- middle order statistic, ``(a + b) / 2`` for an even count.
"""

from __future__ import annotations

import numpy as np

GRAY_WEIGHTS = (0.299, 0.587, 0.114)  # edge_pipeline.py:22
DBL_EPSILON = np.finfo(np.float64).eps


def to_grayscale(image):
    """edge_pipeline.py:42-49: ((0.299 R + 0.587 G) + 0.114 B), clipped to [0, 1]."""
    image = np.asarray(image, dtype=np.float64)
    if image.ndim != 3 or image.shape[2] != 3 or image.shape[0] < 1 or image.shape[1] < 1:
        raise ValueError("expected a non-empty (H, W, 3) image")
    r, g, b = GRAY_WEIGHTS
    acc = r * image[:, :, 0]
    acc = acc + g * image[:, :, 1]
    acc = acc + b * image[:, :, 2]
    return np.clip(acc, 0.0, 1.0)


def blur_kernel_5x5(sigma):
    """edge_pipeline.py:52-59: normalised outer product of 1-D exponentials."""
    if sigma <= 0.0:
        raise ValueError("sigma must be positive")
    d = np.arange(-2, 3, dtype=np.float64)
    k1 = np.exp(-(d * d) / (2.0 * sigma * sigma))
    k2 = np.outer(k1, k1)
    return k2 / k2.sum()


def correlate_nearest(img, weights):
    """NI_Correlate restated: acc = 0; acc += x*w over kept taps, row-major."""
    img = np.asarray(img, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    kh, kw = weights.shape
    rh, rw = kh // 2, kw // 2
    padded = np.pad(img, ((rh, rh), (rw, rw)), mode="edge")
    h, w = img.shape
    acc = np.zeros_like(img)
    for a in range(kh):
        for b in range(kw):
            wt = weights[a, b]
            if not abs(wt) > DBL_EPSILON:
                continue
            acc = acc + padded[a:a + h, b:b + w] * wt
    return acc


def gaussian_blur_5x5(gray, sigma=1.0):
    """edge_pipeline.py:62-67 (convolve == correlate: the kernel is bitwise symmetric)."""
    gray = np.asarray(gray, dtype=np.float64)
    k = blur_kernel_5x5(sigma)
    return np.clip(correlate_nearest(gray, k[::-1, ::-1]), 0.0, 1.0)


SOBEL_X = np.array([[-1.0, 0.0, 1.0], [-2.0, 0.0, 2.0], [-1.0, 0.0, 1.0]])  # :24-26
SOBEL_Y = SOBEL_X.T  # :27


def hypot_glibc(x, y):
    """glibc 2.35+ ``__hypot`` (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel).

    Restated from the libm.so.6 (glibc 2.39) machine code in this image:
    constants LARGE=2^511, TINY=2^-459, EPS=2^-54, SCALE=2^-600.
    """
    x = np.abs(np.asarray(x, dtype=np.float64))
    y = np.abs(np.asarray(y, dtype=np.float64))
    ax = np.maximum(x, y)
    ay = np.minimum(x, y)
    out = np.empty(np.broadcast(ax, ay).shape)
    ax, ay = np.broadcast_arrays(ax, ay)

    def kernel(a, b):
        h = np.sqrt(a * a + b * b)
        big = h <= b + b
        d1 = h - b
        t1a = ((d1 + d1) - a) * a
        t2a = (d1 - ((a - b) + (a - b))) * d1
        d2 = h - a
        t1b = (d2 + d2) * (a - (b + b))
        t2b = ((4.0 * d2) - b) * b + d2 * d2
        t1 = np.where(big, t1a, t1b)
        t2 = np.where(big, t2a, t2b)
        return h - (t1 + t2) / (h + h)

    with np.errstate(all="ignore"):
        large = ax > 2.0 ** 511
        tiny = (~large) & (ay < 2.0 ** -459)
        common = ~(large | tiny)
        trivial = np.where(large, ay <= ax * 2.0 ** -54,
                           np.where(tiny, ax >= ay * 2.0 ** 54, ay <= ax * 2.0 ** -54))
        res = np.where(common, kernel(ax, ay), 0.0)
        res = np.where(large, kernel(ax * 2.0 ** -600, ay * 2.0 ** -600) * 2.0 ** 600, res)
        res = np.where(tiny, kernel(ax * 2.0 ** 600, ay * 2.0 ** 600) * 2.0 ** -600, res)
        res = np.where(trivial, ax + ay, res)
        nonfinite = ~(np.isfinite(ax) & np.isfinite(ay))
        res = np.where(nonfinite, np.where(np.isinf(ax) | np.isinf(ay), np.inf, ax + ay), res)
    out[...] = res
    return out


def sobel_gradients(gray):
    """edge_pipeline.py:70-83: (magnitude, orientation) with edge replication."""
    gray = np.asarray(gray, dtype=np.float64)
    if gray.ndim != 2 or gray.shape[0] < 3 or gray.shape[1] < 3:
        raise ValueError("Sobel gradients need a grayscale image of at least 3x3")
    gx = correlate_nearest(gray, SOBEL_X)
    gy = correlate_nearest(gray, SOBEL_Y)
    mag = np.hypot(gx, gy)
    ori = np.mod(np.arctan2(gy, gx), np.pi)
    return mag, ori


def orientation_bins(ori):
    """edge_pipeline.py:102: floor((theta + pi/8) / (pi/4)) mod 4."""
    return np.floor((ori + np.pi / 8) / (np.pi / 4)).astype(np.int64) % 4


# (prev, next) neighbour offsets per bin, edge_pipeline.py:104-109
NMS_OFFSETS = {0: ((0, -1), (0, 1)), 1: ((-1, -1), (1, 1)),
               2: ((-1, 0), (1, 0)), 3: ((-1, 1), (1, -1))}


def nms_thin(mag, ori):
    """edge_pipeline.py:86-114: keep iff mag > prev and mag >= next; OOB neighbours = 0."""
    mag = np.asarray(mag, dtype=np.float64)
    ori = np.asarray(ori, dtype=np.float64)
    if mag.shape != ori.shape:
        raise ValueError("magnitude and orientation shapes differ")
    h, w = mag.shape
    z = np.zeros((h + 2, w + 2))
    z[1:-1, 1:-1] = mag
    bins = orientation_bins(ori)
    keep = np.zeros((h, w), dtype=bool)
    for b, ((pa, pb), (na, nb)) in NMS_OFFSETS.items():
        prev = z[1 + pa:1 + pa + h, 1 + pb:1 + pb + w]
        nxt = z[1 + na:1 + na + h, 1 + nb:1 + nb + w]
        keep |= (bins == b) & (mag > prev) & (mag >= nxt)
    return np.where(keep, mag, 0.0)


def positive_median(values):
    """np.median of the strictly positive entries; 1.0 when there are none (:123-124)."""
    v = np.asarray(values, dtype=np.float64).ravel()
    pos = v[v > 0.0]
    n = pos.size
    if n == 0:
        return 1.0
    k = (n - 1) // 2
    if n % 2:
        return float(np.partition(pos, k)[k])
    part = np.partition(pos, [k, k + 1])
    return float((part[k] + part[k + 1]) / 2.0)


def median_normalize(thinned):
    """edge_pipeline.py:117-125: min(v / (2 m), 1)."""
    thinned = np.asarray(thinned, dtype=np.float64)
    m = positive_median(thinned)
    return np.minimum(thinned / (2.0 * m), 1.0)


def importance_pipeline(image, sigma=1.0, nms=True, median=True):
    """edge_pipeline.py:128-135 (gray input is not clipped); ``nms``/``median``
    mirror the CLI's ``--no-nms``/``--no-median`` (io_cli.py:315-323)."""
    image = np.asarray(image, dtype=np.float64)
    gray = image if image.ndim == 2 else to_grayscale(image)
    mag, ori = sobel_gradients(gaussian_blur_5x5(gray, sigma))
    out = nms_thin(mag, ori) if nms else mag
    return median_normalize(out) if median else out


def importance_batch(images, sigma=1.0):
    """Per-view pipeline over a (B, H, W, 3) or (B, H, W) stack (per-image medians)."""
    images = np.asarray(images)
    return np.stack([importance_pipeline(im, sigma) for im in images])


def sample_scores(importance, positions):
    """edge_pipeline.py:138-164: bilinear sample at (x, y); outside [0, W-1] x [0, H-1] -> 0.

    value = ((1 - fy) * ((1 - fx) v00 + fx v01)) + (fy * ((1 - fx) v10 + fx v11)), each
    product and sum rounded separately (numpy evaluates the expression left to right).
    NaN positions make numpy index with INT64_MIN: the reference raises IndexError.
    """
    importance = np.asarray(importance, dtype=np.float64)
    positions = np.asarray(positions, dtype=np.float64).reshape(-1, 2)
    h, w = importance.shape
    x, y = positions[:, 0], positions[:, 1]
    if np.isnan(positions).any():
        raise IndexError("NaN sample position")
    inside = (x >= 0.0) & (x <= w - 1.0) & (y >= 0.0) & (y <= h - 1.0)
    xc = np.minimum(np.maximum(x, 0.0), w - 1.0)
    yc = np.minimum(np.maximum(y, 0.0), h - 1.0)
    x0 = np.floor(xc).astype(np.int64)
    y0 = np.floor(yc).astype(np.int64)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    fx = xc - x0
    fy = yc - y0
    top = (1 - fx) * importance[y0, x0] + fx * importance[y0, x1]
    bot = (1 - fx) * importance[y1, x0] + fx * importance[y1, x1]
    value = (1 - fy) * top + fy * bot
    return np.where(inside, value, 0.0)
