"""Drop-in for ``splitkit.densify_controller`` on B200 (3D scenes).

Same names and semantics as ``/root/reference/pkg/src/splitkit/
densify_controller.py``; the statistics live on the device and selection is
one cooperative radix-select launch (``igs_select_candidates``).
``densify_step`` runs select -> LAS pre-pass -> ONE 32-byte device->host read
({eligible, take, n_split, flags}) -> LAS apply, and returns the same
``DensifyEvent`` as the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import las_split as _las
from .core import Scene2, Scene3
from .schedule import DensifyConfig, is_densify_step, is_warmup_step


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_08661_b200 needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


class DensifyStats:
    """Per-primitive selection signals between densify events (densify_controller.py:23-51),
    float64 on the device.

    ``edge_score`` is assignable like the reference's attribute (``stats.edge_score =
    sample_scores(...)``, splat2d.py:397): numpy arrays and tensors of any float dtype on any
    device are converted and copied into the device buffer the kernels read, after a length
    check, so the selection never sees a host pointer, a short buffer or the wrong dtype."""

    def __init__(self, count: int, device=None):
        self._device = torch.device(device) if device is not None else _dev()
        self._new(count)

    def _new(self, count: int):
        # rows: gradient-norm sums, edge scores.  A reset does not fill them: a row marked
        # pending reads as zeros (zeroed on first access), the first position-gradient
        # accumulation stores instead of adding, and an assignment of the edge scores
        # overwrites the row -- so in the trainer's loop the reset's zeros are never written.
        self._buf = torch.empty(2, count, dtype=torch.float64, device=self._device)
        self._pending = [True, True]
        self._accum_count = 0

    def _row(self, k: int) -> torch.Tensor:
        if self._pending[k]:
            self._buf[k].zero_()
            self._pending[k] = False
        return self._buf[k]

    @property
    def _grad_sum(self) -> torch.Tensor:
        return self._row(0)

    def _ptr(self, k: int) -> int:
        """Device address of row k (0: gradient sums, 1: edge scores) for the kernels, zeroed
        first if pending (no tensor view built on the launch path)."""
        if self._pending[k]:
            self._buf[k].zero_()
            self._pending[k] = False
        return self._buf.data_ptr() + k * self._buf.stride(0) * 8

    def __len__(self):
        return self._buf.shape[1]

    @property
    def grad_norm(self):
        if self._accum_count == 0:
            return torch.zeros(len(self), dtype=torch.float64, device=self._device)
        return self._grad_sum / self._accum_count

    @property
    def edge_score(self):
        return self._row(1)

    @edge_score.setter
    def edge_score(self, values):
        v = values if isinstance(values, torch.Tensor) else torch.as_tensor(np.asarray(values))
        if v.dtype == torch.bool or v.is_complex():
            raise TypeError(f"edge scores must be real numbers, got {v.dtype}")
        if v.ndim != 1 or v.shape[0] != len(self):
            raise ValueError(f"edge score length {tuple(v.shape)} does not match stats length "
                             f"({len(self)},)")
        self._buf[1].copy_(v.to(self._device, torch.float64))
        self._pending[1] = False

    def reset(self, count: int | None = None):
        """Fresh zero statistics (new buffers, as the reference's new arrays; no fill kernel)."""
        self._new(len(self) if count is None else count)

    def set_edge_score(self, values):
        self.edge_score = values


def accumulate_grads(stats: DensifyStats, step_grad_norms) -> DensifyStats:
    """Fold one iteration's gradient norms into the running mean (densify_controller.py:54-63)."""
    x = step_grad_norms
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float64))
    t = t.to(stats._device, torch.float64)
    if tuple(t.shape) != tuple(stats._grad_sum.shape):
        raise ValueError(f"gradient norms length {tuple(t.shape)} does not match stats length "
                         f"{tuple(stats._grad_sum.shape)}")
    stats._grad_sum.add_(t)
    stats._accum_count += 1
    return stats


def accumulate_position_grads(stats: DensifyStats, grad_xy) -> DensifyStats:
    """accumulate_grads(stats, np.hypot(g[:, 0], g[:, 1])) fused on the device
    (splat2d.py:393-394): one kernel adds glibc-exact float64 hypot of each primitive's (x, y)
    positional gradient to its running sum."""
    g = grad_xy if isinstance(grad_xy, torch.Tensor) else torch.as_tensor(np.asarray(grad_xy))
    if g.dtype not in (torch.float32, torch.float64):
        g = g.to(torch.float64)
    g = g.to(stats._device).contiguous()
    if g.ndim != 2 or g.shape[1] != 2 or g.shape[0] != len(stats):
        raise ValueError(f"positional gradients {tuple(g.shape)} do not match stats length "
                         f"{len(stats)} (need (N, 2))")
    L = _lib.lib()
    dtype = _lib.IGS_F64 if g.dtype == torch.float64 else _lib.IGS_F32
    if stats._pending[0]:                 # first accumulation since the reset: store 0.0 + h
        dtype |= _lib.IGS_ACCUM_STORE
    _lib.check(L.igs_accumulate_grad_norms(stats._buf[0].data_ptr(), g.data_ptr(), dtype,
                                           len(stats), _lib.stream_handle()), "accumulate_grads")
    stats._pending[0] = False
    stats._accum_count += 1
    return stats


def _take_cap(cfg: DensifyConfig, count: int, headroom: int) -> int:
    """min(headroom, max(ceil(growth_cap*count - 1e-9), 0)) (densify_controller.py:99-100)."""
    cap = math.ceil(cfg.growth_cap * count - 1e-9)
    return min(headroom, max(cap, 0))


def _launch_select(stats: DensifyStats, cfg: DensifyConfig, step: int, take_cap: int,
                   counts=None):
    """Async select; returns (mask uint8 tensor, counts int64[2] device tensor). ``counts``
    (optional) is the device int64[2] to write {#eligible, take} into."""
    n = len(stats)
    L = _lib.lib()
    mask = torch.empty(n, dtype=torch.uint8, device=stats._device)
    if counts is None:
        counts = torch.empty(2, dtype=torch.int64, device=stats._device)  # the kernel writes both
    nbytes = _lib.query_size(L.igs_select_workspace_bytes, n)
    ws = _lib.workspace(nbytes, stats._device, "select")
    _lib.check(L.igs_select_candidates(
        stats._ptr(0), stats._accum_count, stats._ptr(1), n,
        float(cfg.grad_threshold), int(is_warmup_step(cfg, step)), _lib.IGS_POLICY[cfg.policy],
        int(take_cap), mask.data_ptr(), counts.data_ptr(), ws.data_ptr(), ws.numel(),
        _lib.stream_handle()), "select_candidates")
    return mask, counts


def select_candidates(stats: DensifyStats, cfg: DensifyConfig, step: int, headroom: int):
    """Boolean mask (CUDA tensor) of the primitives to split (densify_controller.py:80-106)."""
    if headroom < 0:
        raise ValueError("headroom must be non-negative")
    n = len(stats)
    if headroom == 0 or n == 0:
        return torch.zeros(n, dtype=torch.bool, device=stats._device)
    take_cap = _take_cap(cfg, n, headroom)
    if take_cap <= 0:
        return torch.zeros(n, dtype=torch.bool, device=stats._device)
    mask, _ = _launch_select(stats, cfg, step, take_cap)
    return mask.view(torch.bool)


def eligible_count(stats: DensifyStats, cfg: DensifyConfig, step: int) -> int:
    """int(_eligible_mask(stats, cfg, step).sum()) (densify_controller.py:66-69)."""
    if is_warmup_step(cfg, step):
        return len(stats)
    return int((stats.grad_norm > cfg.grad_threshold).sum())


@dataclass(frozen=True)
class DensifyEvent:
    """What one densify event did: step, eligible count, splits, count after (densify_controller.py:109-119)."""

    step: int
    eligible: int
    split: int
    count_after: int

    def as_csv_row(self) -> str:
        return f"{self.step},{self.eligible},{self.split},{self.count_after}"


EVENT_CSV_HEADER = "step,eligible,split,count_after"


def densify_step(scene, stats: DensifyStats, cfg: DensifyConfig, step: int) -> DensifyEvent:
    """One densify event on a GPU 3D scene, in place (densify_controller.py:125-147)."""
    if not is_densify_step(cfg, step):
        raise ValueError(f"step {step} is not a densify step for this timetable")
    if len(stats) != scene.count:
        raise ValueError("stats length does not match scene count")
    if not isinstance(scene, (Scene2, Scene3)):
        raise TypeError(f"unsupported scene type {type(scene).__name__}")
    headroom = scene.capacity - scene.count
    n = scene.count
    take_cap = _take_cap(cfg, n, headroom) if (headroom > 0 and n > 0) else 0
    c = cfg.split_constants
    if take_cap > 0:
        # select, then the fused split (pre-pass + device-guarded apply); one host read
        # counts | split summary, written by the kernels straight into pinned host memory
        res, view = _las.pinned_summary(stats._device, 4)
        view[0] = view[3] = -1  # unwritten: the select's eligible count, the split's flags
        mask, _ = _launch_select(stats, cfg, step, take_cap, counts=res[:2])
        _las.split_async(scene, mask.view(torch.bool), c, summary=res[2:],
                         sparse=4 * take_cap <= n)  # at most a quarter masked: list mode
        # the apply pass may still run: the statistics reset below is ordered after it
        _las.wait_summary(stats._device, res[2:])
        _las.wait_word(stats._device, res, 0)
        eligible, n_split, flags = int(view[0]), int(view[2]), int(view[3])
        _las.finish_split(scene, n_split, flags)
    else:
        eligible, n_split = eligible_count(stats, cfg, step), 0
    stats.reset(scene.count)
    return DensifyEvent(step=step, eligible=eligible, split=n_split, count_after=scene.count)
