"""ctypes binding of libigs_b200.so (include/igs_b200.h) plus workspace/stream plumbing.

The product path has no CPU fallback: if the shared library or a CUDA device
is missing, every entry point raises ``RuntimeError`` naming what is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IGS_LIB") or os.path.join(HERE, "libigs_b200.so")  # IGS_LIB: A/B runs

IGS_OK, IGS_ERR_ARGUMENT, IGS_ERR_CUDA, IGS_ERR_WORKSPACE, IGS_ERR_UNSUPPORTED = range(5)
IGS_F32, IGS_F64 = 0, 1
IGS_ACCUM_STORE = 0x100  # igs_accumulate_grad_norms: store 0.0 + h (first accumulation)
IGS_EDGE_NO_NMS, IGS_EDGE_NO_MEDIAN = 1, 2
IGS_POLICY = {"product": 0, "edge": 1, "grad": 2}
IGS_LAS_BAD_QUAT, IGS_LAS_BAD_OPACITY, IGS_LAS_RENORM = 1, 2, 4
IGS_SHARD_HIST_LEN = 65537  # include/igs_b200.h

_vp, _i64, _sz, _int, _dbl, _flt = C.c_void_p, C.c_int64, C.c_size_t, C.c_int, C.c_double, C.c_float
_szp = C.POINTER(C.c_size_t)

# name -> (restype, argtypes); the exported C ABI, one line per include/igs_b200.h symbol
SIGNATURES = {
    "igs_strerror": (C.c_char_p, [_int]),
    "igs_last_cuda_error": (C.c_char_p, []),
    "igs_abi_version": (_int, []),
    "igs_stream_synchronize": (_int, [_vp]),
    "igs_wait_host_word": (_int, [_vp, _i64, _i64, _vp]),
    "igs_publish_words": (_int, [_vp, _vp, _i64, _vp]),
    "igs_l2_set_aside": (_int, [_sz, _szp]),
    "igs_edge_workspace_bytes": (_int, [_i64, _i64, _i64, _int, _szp]),
    "igs_edge_importance": (_int, [_vp, _int, _int, _i64, _i64, _i64, _vp, _int, _vp, _vp, _sz,
                                   _vp]),
    "igs_to_grayscale": (_int, [_vp, _int, _i64, _i64, _i64, _vp, _vp]),
    "igs_gaussian_blur_5x5": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "igs_sobel_gradients": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "igs_nms_thin": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "igs_median_normalize": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "igs_normalize_quaternions": (_int, [_vp, _i64, _vp, _vp]),
    "igs_sample_scores": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp]),
    "igs_debug_edge_trace": (_int, [_vp, _i64, C.POINTER(C.c_int64)]),
    "igs_debug_edge_phases": (_int, [_vp, _int]),
    "igs_select_workspace_bytes": (_int, [_i64, _szp]),
    "igs_select_candidates": (_int, [_vp, _i64, _vp, _i64, _dbl, _int, _int, _i64, _vp, _vp, _vp,
                                     _sz, _vp]),
    "igs_accumulate_grad_norms": (_int, [_vp, _vp, _int, _i64, _vp]),
    "igs_shard_workspace_bytes": (_int, [_i64, _szp]),
    "igs_shard_keys": (_int, [_vp, _i64, _vp, _i64, _dbl, _int, _int, _vp, _vp, _sz, _vp]),
    "igs_shard_boundary": (_int, [_vp, _i64, _vp, _vp, _vp, _flt, _i64, _i64, _vp, _vp, _vp,
                                  _sz, _vp]),
    "igs_shard_finalize": (_int, [_vp, _int, _int, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _sz,
                                  _vp]),
    "igs_shard_child_index": (_int, [_vp, _i64, _vp, _vp]),
    "igs_shard_mask": (_int, [_vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "igs_las_workspace_bytes": (_int, [_i64, _szp]),
    "igs_las_prepare": (_int, [_vp, _vp, _vp, _i64, _flt, _vp, _sz, _vp, _vp]),
    "igs_las_apply": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _flt, _flt, _flt,
                             _flt, _int, _vp, _sz, _vp]),
    "igs_las_split": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _flt, _flt, _flt,
                             _flt, _vp, _sz, _vp, _vp]),
    "igs_las_split_packed": (_int, [_vp]),
    "igs_shard_event": (_int, [_vp]),
    "igs_las_split_sparse": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _flt, _flt,
                                    _flt, _flt, _vp, _sz, _vp, _vp]),
    "igs_las2d_split": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _flt, _flt, _flt, _flt,
                               _vp, _sz, _vp, _vp]),
    "igs_las2d_apply": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _flt, _flt, _flt, _flt,
                               _vp, _sz, _vp]),
    "igs_las_split_guarded": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _int, _i64, _i64, _vp, _flt,
                                     _flt, _flt, _flt, _vp, _vp, _sz, _vp]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and type the C ABI.  Works without a GPU (symbol checks only)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"{path} is missing: build it with `python -m paper_2603_08661_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype, fn.argtypes = res, args
            _lib = lib
    return _lib


_cuda_ok = False


def lib():
    """The library, after checking (once) that a CUDA device is present."""
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2603_08661_b200 needs a CUDA device (sm_100a); "
                               "there is no CPU fallback")
        _cuda_ok = True
    return _lib if _lib is not None else load()


def check(status: int, what: str):
    if status == IGS_OK:
        return
    L = load()
    msg = L.igs_strerror(status).decode()
    if status == IGS_ERR_CUDA:
        msg += f" ({L.igs_last_cuda_error().decode()})"
    if status == IGS_ERR_ARGUMENT:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


try:  # the raw cudaStream_t of the current stream without building a Stream object
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover - older torch
    _raw_stream = None


class LasSplitArgs(C.Structure):
    """Mirror of IgsLasSplitArgs (include/igs_b200.h)."""
    _fields_ = [("positions", _vp), ("log_scales", _vp), ("rotations", _vp),
                ("opacity_logits", _vp), ("sh", _vp), ("sh_floats", _i64), ("count", _i64),
                ("capacity", _i64), ("mask", _vp), ("alpha", _flt), ("log_alpha", _flt),
                ("log_gamma", _flt), ("beta", _flt), ("workspace", _vp),
                ("workspace_bytes", _sz), ("summary", _vp), ("stream", _vp),
                ("sparse", C.c_int32), ("reserved", C.c_int32)]


class ShardEventArgs(C.Structure):
    """Mirror of IgsShardEventArgs (include/igs_b200.h)."""
    _fields_ = [("records", _vp), ("world", C.c_int32), ("rank", C.c_int32),
                ("record_cap", _i64), ("n_global", _i64), ("gidx", _vp), ("n", _i64),
                ("mask", _vp), ("plan", _vp), ("shard_workspace", _vp),
                ("shard_workspace_bytes", _sz), ("host_plan", _vp), ("plan_words", _i64),
                ("split", C.c_int32), ("dims", C.c_int32), ("positions", _vp),
                ("log_scales", _vp), ("rotations", _vp), ("opacity_logits", _vp),
                ("sh_or_colors", _vp), ("sh_floats", _i64), ("reserved_rows", _i64),
                ("alpha", _flt), ("log_alpha", _flt), ("log_gamma", _flt), ("beta", _flt),
                ("las_workspace", _vp), ("las_workspace_bytes", _sz), ("stream", _vp)]


def stream_handle(device=None) -> int:
    if _raw_stream is not None:
        idx = torch.cuda.current_device() if device is None else torch.device(device).index
        if idx is None:
            idx = torch.cuda.current_device()
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


_ws: dict = {}


def workspace(nbytes: int, device, tag: str) -> torch.Tensor:
    """Caller-owned scratch (the library never allocates), cached per (device, stream, tag)."""
    device = torch.device(device)
    key = (device.index, stream_handle(device), tag)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
        _ws[key] = buf
    return buf


_sizes = {}


def query_size(fn, *args) -> int:
    """A *_workspace_bytes query (pure host arithmetic), memoised per (entry point, shape)."""
    key = (fn.__name__, args)
    v = _sizes.get(key)
    if v is None:
        out = C.c_size_t(0)
        check(fn(*args, C.byref(out)), fn.__name__)
        v = _sizes[key] = int(out.value)
    return v
