"""Drop-in for ``splitkit.edge_pipeline`` on B200 (sm_100a).

Same names, arguments, defaults and exceptions as
``/root/reference/pkg/src/splitkit/edge_pipeline.py``; the arithmetic runs in
``libigs_b200.so``.  Inputs may be numpy arrays (copied to the current CUDA
device; results come back as numpy float64 arrays, like the reference) or
torch tensors (CUDA results on the same device).

``importance_pipeline`` is ONE fused persistent kernel launch (gray -> blur ->
Sobel -> NMS -> per-view median histogram -> radix select -> normalise);
``importance_batch`` is the batched form (B views, per-view medians).  The
stage functions are separate kernels, kept for the stage-level API
(``io_cli.py:315-323`` uses them for ``--no-nms`` / ``--no-median``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

GRAY_WEIGHTS = (0.299, 0.587, 0.114)  # Rec.601 luma, edge_pipeline.py:22

SOBEL_X = np.array([[-1.0, 0.0, 1.0],
                    [-2.0, 0.0, 2.0],
                    [-1.0, 0.0, 1.0]])
SOBEL_Y = SOBEL_X.T


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_08661_b200 needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _as_cuda(x, float_ok=(torch.float64,)):
    """(contiguous CUDA tensor, came_from_numpy).  Non-float inputs become float64."""
    if isinstance(x, torch.Tensor):
        t = x
        from_numpy = False
        if not t.is_cuda:
            t = t.to(_device())
    else:
        a = np.asarray(x)
        from_numpy = True
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(_device())
    if t.dtype not in float_ok:
        t = t.to(torch.float64)
    return t.contiguous(), from_numpy


def _ret(t: torch.Tensor, to_numpy: bool):
    return t.cpu().numpy() if to_numpy else t


@dataclass
class GradientField:
    """Sobel output: magnitude and orientation mod pi, same shape (edge_pipeline.py:30-39)."""

    magnitude: object
    orientation: object

    def __post_init__(self):
        if tuple(self.magnitude.shape) != tuple(self.orientation.shape):
            raise ValueError("magnitude and orientation shapes differ")


def to_grayscale(image):
    """Gray image from RGB with the Rec.601 weights, clipped to [0, 1] (edge_pipeline.py:42-49)."""
    img, np_out = _as_cuda(image, (torch.float32, torch.float64))
    if img.ndim != 3 or img.shape[2] != 3 or img.shape[0] < 1 or img.shape[1] < 1:
        raise ValueError("expected a non-empty (H, W, 3) image")
    h, w = img.shape[:2]
    out = torch.empty((h, w), dtype=torch.float64, device=img.device)
    L = _lib.lib()
    _lib.check(L.igs_to_grayscale(img.data_ptr(), _dtype_code(img), 1, h, w, out.data_ptr(),
                                  _lib.stream_handle()), "to_grayscale")
    return _ret(out, np_out)


def blur_kernel_5x5(sigma: float) -> np.ndarray:
    """Normalised 5x5 Gaussian kernel (edge_pipeline.py:52-59), computed on the host so the
    weights are bit-identical to the reference's."""
    if sigma <= 0.0:
        raise ValueError("sigma must be positive")
    offsets = np.arange(-2, 3, dtype=np.float64)
    k1 = np.exp(-(offsets ** 2) / (2.0 * sigma * sigma))
    kernel = np.outer(k1, k1)
    return kernel / kernel.sum()


def _weights(sigma):
    return np.ascontiguousarray(blur_kernel_5x5(sigma), dtype=np.float64)


def _dtype_code(t):
    return _lib.IGS_F64 if t.dtype == torch.float64 else _lib.IGS_F32


def gaussian_blur_5x5(gray, sigma: float = 1.0):
    """5x5 Gaussian blur, edge-replicated borders, clipped to [0, 1] (edge_pipeline.py:62-67)."""
    w = _weights(sigma)
    g, np_out = _as_cuda(gray)
    if g.ndim != 2 or g.shape[0] < 1 or g.shape[1] < 1:
        raise ValueError("gaussian_blur_5x5 expects a non-empty 2-D image")
    out = torch.empty_like(g)
    L = _lib.lib()
    _lib.check(L.igs_gaussian_blur_5x5(g.data_ptr(), 1, g.shape[0], g.shape[1],
                                       w.ctypes.data, out.data_ptr(), _lib.stream_handle()),
               "gaussian_blur_5x5")
    return _ret(out, np_out)


def sobel_gradients(gray) -> GradientField:
    """Sobel magnitude (glibc hypot, bit-exact) and orientation atan2(Gy,Gx) mod pi
    (edge_pipeline.py:70-83).  The image must be at least 3x3."""
    g, np_out = _as_cuda(gray)
    if g.ndim != 2 or g.shape[0] < 3 or g.shape[1] < 3:
        raise ValueError("Sobel gradients need a grayscale image of at least 3x3")
    mag, ori = torch.empty_like(g), torch.empty_like(g)
    L = _lib.lib()
    _lib.check(L.igs_sobel_gradients(g.data_ptr(), 1, g.shape[0], g.shape[1], mag.data_ptr(),
                                     ori.data_ptr(), _lib.stream_handle()), "sobel_gradients")
    return GradientField(_ret(mag, np_out), _ret(ori, np_out))


def nms_thin(field: GradientField):
    """Non-maximum suppression along the quantised gradient direction (edge_pipeline.py:86-114):
    keep iff magnitude > the preceding neighbour and >= the following one; OOB = 0."""
    mag, np_out = _as_cuda(field.magnitude)
    ori, _ = _as_cuda(field.orientation)
    if mag.shape != ori.shape:
        raise ValueError("magnitude and orientation shapes differ")
    if mag.ndim != 2:
        raise ValueError("nms_thin expects 2-D fields")
    out = torch.empty_like(mag)
    if mag.numel():
        L = _lib.lib()
        _lib.check(L.igs_nms_thin(mag.data_ptr(), ori.data_ptr(), 1, mag.shape[0], mag.shape[1],
                                  out.data_ptr(), _lib.stream_handle()), "nms_thin")
    return _ret(out, np_out)


def median_normalize(thinned, medians=None):
    """min(v / (2 * median of positives), 1); median := 1 without positives (:117-125).
    Any shape.  ``medians`` (optional CUDA float64 tensor of shape (1,)) receives m."""
    t, np_out = _as_cuda(thinned)
    out = torch.empty_like(t)
    if t.numel():
        _median_normalize_batched(t.reshape(1, -1), out.reshape(1, -1), medians)
    return _ret(out, np_out)


def _median_normalize_batched(src2d, dst2d, medians=None):
    b, n = src2d.shape
    L = _lib.lib()
    nbytes = _lib.query_size(L.igs_edge_workspace_bytes, b, 1, n, 0)
    ws = _lib.workspace(nbytes, src2d.device, "edge")
    _lib.check(L.igs_median_normalize(src2d.data_ptr(), b, n, dst2d.data_ptr(),
                                      _lib.ptr(medians), ws.data_ptr(), ws.numel(),
                                      _lib.stream_handle()), "median_normalize")


def _edge_launch(img, channels, b, h, w, sigma, flags, out):
    L = _lib.lib()
    wts = _weights(sigma)
    nbytes = _lib.query_size(L.igs_edge_workspace_bytes, b, h, w, flags)
    ws = _lib.workspace(nbytes, img.device, "edge")
    _lib.check(L.igs_edge_importance(img.data_ptr(), _dtype_code(img), channels, b, h, w,
                                     wts.ctypes.data, flags, out.data_ptr(), ws.data_ptr(),
                                     ws.numel(), _lib.stream_handle()), "importance_pipeline")


def importance_pipeline(image, sigma: float = 1.0, *, nms: bool = True, median: bool = True):
    """Full importance map (edge_pipeline.py:128-135): grayscale (skipped, and not clipped, for
    an (H, W) input), blur, Sobel, NMS, median normalisation -- one fused launch.
    ``nms`` / ``median`` = False mirror the CLI's --no-nms / --no-median."""
    img, np_out = _as_cuda(image, (torch.float32, torch.float64))
    if img.ndim == 2:
        channels, (h, w) = 1, img.shape
    else:
        if img.ndim != 3 or img.shape[2] != 3 or img.shape[0] < 1 or img.shape[1] < 1:
            raise ValueError("expected a non-empty (H, W, 3) image")
        channels, (h, w) = 3, img.shape[:2]
    if h < 3 or w < 3:
        raise ValueError("Sobel gradients need a grayscale image of at least 3x3")
    _blur_sigma_check(sigma)
    out = torch.empty((h, w), dtype=torch.float64, device=img.device)
    flags = (0 if nms else _lib.IGS_EDGE_NO_NMS) | (0 if median else _lib.IGS_EDGE_NO_MEDIAN)
    _edge_launch(img, channels, 1, h, w, sigma, flags, out)
    return _ret(out, np_out)


def _blur_sigma_check(sigma):
    if sigma <= 0.0:
        raise ValueError("sigma must be positive")


def importance_batch(images, sigma: float = 1.0, *, out=None, nms: bool = True,
                     median: bool = True, chunk: int = 8):
    """Batched importance maps with per-view medians: (B, H, W, 3) RGB or (B, H, W) gray,
    float32 or float64 -> (B, H, W) float64.  Equal to stacking importance_pipeline(view).

    CUDA input: one fused launch over the whole batch, result on the device.
    Host input (numpy array or CPU tensor; pin it for full PCIe bandwidth): streamed through
    the GPU in chunks of ``chunk`` views with the host->device copy of chunk i+1, the fused
    kernel on chunk i and the device->host copy of chunk i-1 overlapped on three streams;
    the result comes back on the host (numpy for numpy input, else a CPU tensor / ``out``).
    """
    _blur_sigma_check(sigma)
    on_host = not (isinstance(images, torch.Tensor) and images.is_cuda)
    if on_host:
        return _importance_batch_host(images, sigma, out, nms, median, chunk)
    img, np_out = _as_cuda(images, (torch.float32, torch.float64))
    channels, (b, h, w) = _batch_geometry(img)
    if out is None:
        out = torch.empty((b, h, w), dtype=torch.float64, device=img.device)
    elif tuple(out.shape) != (b, h, w) or out.dtype != torch.float64 or not out.is_cuda:
        raise ValueError("out must be a CUDA float64 tensor of shape (B, H, W)")
    flags = (0 if nms else _lib.IGS_EDGE_NO_NMS) | (0 if median else _lib.IGS_EDGE_NO_MEDIAN)
    if b:
        _edge_launch(img, channels, b, h, w, sigma, flags, out)
    return _ret(out, np_out)


def sample_scores(importance, positions, view=None):
    """Importance at (x, y) pixel positions by bilinear interpolation (edge_pipeline.py:138-164);
    positions outside [0, W-1] x [0, H-1] score 0.  Batched form: ``importance`` (B, H, W) and
    ``view`` (N,) int map indices.  numpy in -> numpy out; CUDA tensors -> CUDA tensor."""
    imp, np_out = _as_cuda(importance)
    pos, _ = _as_cuda(positions)
    if imp.ndim == 2:
        imp = imp.unsqueeze(0)
    if imp.ndim != 3:
        raise ValueError("importance must be (H, W) or (B, H, W)")
    pos = pos.reshape(-1, 2).contiguous()
    if pos.data_ptr() % 16:
        pos = pos.clone()
    n = pos.shape[0]
    vw = None
    if view is not None:
        vw = torch.as_tensor(np.asarray(view) if not isinstance(view, torch.Tensor) else view)
        vw = vw.to(imp.device, torch.int32).reshape(-1).contiguous()
        if vw.shape[0] != n:
            raise ValueError("view must have one entry per position")
    elif imp.shape[0] != 1:
        raise ValueError("batched importance maps need a view index per position")
    out = torch.empty(n, dtype=torch.float64, device=imp.device)
    flags = torch.zeros(1, dtype=torch.int32, device=imp.device)
    L = _lib.lib()
    _lib.check(L.igs_sample_scores(imp.data_ptr(), imp.shape[0], imp.shape[1], imp.shape[2],
                                   pos.data_ptr(), _lib.ptr(vw), n, out.data_ptr(),
                                   flags.data_ptr(), _lib.stream_handle()), "sample_scores")
    f = int(flags.item()) if n else 0
    if f & 1:
        raise IndexError("NaN sample position (the reference indexes with INT64_MIN)")
    if f & 2:
        raise IndexError("view index out of range")
    return _ret(out, np_out)


def _batch_geometry(img):
    if img.ndim == 4:
        if img.shape[3] != 3:
            raise ValueError("expected (B, H, W, 3) RGB views or (B, H, W) gray views")
        channels = 3
    elif img.ndim == 3:
        channels = 1
    else:
        raise ValueError("expected (B, H, W, 3) RGB views or (B, H, W) gray views")
    b, h, w = img.shape[:3]
    if h < 3 or w < 3:
        raise ValueError("Sobel gradients need a grayscale image of at least 3x3")
    return channels, (b, h, w)


_STREAMS: dict = {}


def _pipeline_streams(dev):
    key = dev.index
    if key not in _STREAMS:
        _STREAMS[key] = tuple(torch.cuda.Stream(dev) for _ in range(3))
    return _STREAMS[key]


def _importance_batch_host(images, sigma, out, nms, median, chunk):
    np_in = not isinstance(images, torch.Tensor)
    if np_in:
        a = np.asarray(images)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        src = torch.from_numpy(np.ascontiguousarray(a))
    else:
        src = images.contiguous()
        if src.dtype not in (torch.float32, torch.float64):
            src = src.to(torch.float64)
    channels, (b, h, w) = _batch_geometry(src)
    if out is None:
        res = torch.empty((b, h, w), dtype=torch.float64, pin_memory=src.is_pinned())
    else:
        res = out if isinstance(out, torch.Tensor) else torch.from_numpy(out)
        if tuple(res.shape) != (b, h, w) or res.dtype != torch.float64 or res.is_cuda:
            raise ValueError("out must be a host float64 array of shape (B, H, W)")
    dev = _device()
    flags = (0 if nms else _lib.IGS_EDGE_NO_NMS) | (0 if median else _lib.IGS_EDGE_NO_MEDIAN)
    chunk = max(1, min(int(chunk), b)) if b else 1
    nbuf = 2
    d_in = [torch.empty((chunk,) + tuple(src.shape[1:]), dtype=src.dtype, device=dev)
            for _ in range(nbuf)]
    d_out = [torch.empty((chunk, h, w), dtype=torch.float64, device=dev) for _ in range(nbuf)]
    s_h2d, s_cmp, s_d2h = _pipeline_streams(dev)
    cur = torch.cuda.current_stream(dev)
    for s in (s_h2d, s_cmp, s_d2h):
        s.wait_stream(cur)
    ev_in_free = [None] * nbuf    # compute finished reading d_in[k]
    ev_out_free = [None] * nbuf   # D2H finished reading d_out[k]
    for i, v0 in enumerate(range(0, b, chunk)):
        k, n = i % nbuf, min(chunk, b - v0)
        with torch.cuda.stream(s_h2d):
            if ev_in_free[k] is not None:
                s_h2d.wait_event(ev_in_free[k])
            d_in[k][:n].copy_(src[v0:v0 + n], non_blocking=True)
            ev_loaded = torch.cuda.Event()
            ev_loaded.record(s_h2d)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_loaded)
            if ev_out_free[k] is not None:
                s_cmp.wait_event(ev_out_free[k])
            _edge_launch(d_in[k], channels, n, h, w, sigma, flags, d_out[k])
            ev_done = torch.cuda.Event()
            ev_done.record(s_cmp)
            ev_in_free[k] = ev_done
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_done)
            res[v0:v0 + n].copy_(d_out[k][:n], non_blocking=True)
            ev_o = torch.cuda.Event()
            ev_o.record(s_d2h)
            ev_out_free[k] = ev_o
    for s in (s_h2d, s_cmp, s_d2h):
        cur.wait_stream(s)
    for t in d_in + d_out:
        t.record_stream(cur)
    torch.cuda.current_stream(dev).synchronize()
    if np_in and out is None:
        return res.numpy()
    return out if out is not None else res
