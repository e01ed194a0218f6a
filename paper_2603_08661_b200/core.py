"""Device-resident Gaussian scenes for the densification path.

``Scene3`` mirrors ``splitkit.core.Scene3`` (``/root/reference/pkg/src/splitkit/
core.py:122-200``): the same column names (``positions``, ``log_scales``,
``rotations``, ``opacity_logits``, ``colors``), ``count``, ``capacity``,
``validate``, ``copy``, ``empty``.  B200 layout differences:

* storage is pre-reserved on the GPU (float32 SoA), so a split appends children
  in place instead of re-allocating every column (``_append_columns``,
  core.py:151-157, is an O(N) copy per split);
* spherical harmonics: ``sh`` is a (rows, K, 3) block whose first coefficient
  triplet IS ``colors`` (K = 1 is the reference's colour-only scene, K = 16 is
  SH degree 3); rows of 48 floats are 16-byte aligned so the split clones them
  with 16-byte vector copies.

Attribute semantics the reference's callers rely on:

* reading a column returns a device view of the first ``count`` rows;
* assigning a column (``scene.positions = new``, the trainer's update idiom,
  ``splat2d.py:382-391``) copies the values into the device storage; the new
  column must have ``count`` rows;
* ``capacity`` is assignable (``io_cli.py:339-343`` does ``scene.capacity =
  budget``); raising it past the reserved rows re-reserves the storage and
  keeps the live rows, so the value the kernels see never exceeds the
  allocation.
"""

from __future__ import annotations

import numpy as np
import torch


def _dev(device):
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_08661_b200 needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _as_tensor(x):
    return x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))


def _col(x, n_cols, dtype, device):
    t = _as_tensor(x).to(device=device, dtype=dtype)
    return t.reshape(-1, n_cols) if n_cols else t.reshape(-1)


class _Column:
    """A scene column: ``count`` rows of the reserved buffer ``scene.<attr>``.  ``dc`` selects
    the first SH triplet (the reference's ``colors``) of a (rows, K, 3) block."""

    def __init__(self, attr, dc=False):
        self.attr, self.dc = attr, dc

    def __set_name__(self, owner, name):
        self.name = name

    def _view(self, obj):
        v = getattr(obj, self.attr)[: obj._count]
        return v[:, 0, :] if self.dc else v

    def __get__(self, obj, objtype=None):
        if obj is None:
            return self
        return self._view(obj)

    def __set__(self, obj, value):
        dst = self._view(obj)
        t = _as_tensor(value)
        if t.numel() != dst.numel() or (t.ndim >= 1 and t.shape[0] != obj._count):
            raise ValueError(
                f"column {self.name}: got shape {tuple(t.shape)}, the scene holds {obj._count} "
                f"rows of shape {tuple(dst.shape[1:])} (a device scene keeps one count for "
                "every column; grow it with a split)")
        dst.copy_(t.to(device=dst.device, dtype=dst.dtype).reshape(dst.shape))


class _DeviceScene:
    """Shared storage logic: ``_buffers`` names the reserved per-column buffers (leading
    dimension = reserved rows); ``capacity`` never exceeds the reserved rows."""

    _buffers: tuple = ()

    @property
    def count(self) -> int:
        return self._count

    @property
    def capacity(self) -> int:
        return self._capacity

    @capacity.setter
    def capacity(self, value):
        value = int(value)
        if value < 1:
            raise ValueError("capacity must be positive")
        if value > self.reserved_rows:
            self._reserve(value)
        self._capacity = value

    @property
    def reserved_rows(self) -> int:
        return getattr(self, self._buffers[0]).shape[0]

    def _reserve(self, rows: int):
        """Re-reserve every buffer at `rows` rows, keeping the live rows (stream-ordered)."""
        n = self._count
        for attr in self._buffers:
            old = getattr(self, attr)
            new = torch.empty((rows,) + tuple(old.shape[1:]), dtype=old.dtype, device=old.device)
            new[:n] = old[:n]
            setattr(self, attr, new)

    def validate(self):
        if self._count > self._capacity:
            raise ValueError(f"count {self._count} exceeds capacity {self._capacity}")
        return self

    def _set_count(self, n: int):
        if n > self._capacity or n > self.reserved_rows:
            raise ValueError(f"count {n} exceeds capacity {self._capacity}")
        self._count = int(n)


class Scene3(_DeviceScene):
    """GPU structure-of-arrays 3D scene with pre-reserved capacity."""

    _columns = ("positions", "log_scales", "rotations", "opacity_logits", "colors")
    _buffers = ("_pos", "_ls", "_rot", "_op", "_sh")

    positions = _Column("_pos")
    log_scales = _Column("_ls")
    rotations = _Column("_rot")
    opacity_logits = _Column("_op")
    colors = _Column("_sh", dc=True)
    sh = _Column("_sh")

    def __init__(self, positions, log_scales, rotations, opacity_logits, colors, capacity,
                 dtype=np.float32, device=None):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        if np.dtype(dtype) != np.float32:
            raise ValueError("the B200 scene stores float32 columns")
        dev = _dev(device)
        f = torch.float32
        pos = _col(positions, 3, f, dev)
        ls = _col(log_scales, 3, f, dev)
        rot = _col(rotations, 4, f, dev)
        op = _col(opacity_logits, 0, f, dev)
        c = _as_tensor(colors).to(device=dev, dtype=f)
        sh = c if c.ndim == 3 else c.reshape(-1, 1, 3)
        n = pos.shape[0]
        for name, col in (("log_scales", ls), ("rotations", rot), ("opacity_logits", op),
                          ("colors", sh)):
            if col.shape[0] != n:
                raise ValueError(f"column {name} has length {col.shape[0]} != {n}")
        cap = int(capacity)
        if n > cap:
            raise ValueError(f"count {n} exceeds capacity {cap}")
        self._capacity = cap
        self._pos = torch.empty((cap, 3), dtype=f, device=dev)
        self._ls = torch.empty((cap, 3), dtype=f, device=dev)
        self._rot = torch.empty((cap, 4), dtype=f, device=dev)
        self._op = torch.empty((cap,), dtype=f, device=dev)
        self._sh = torch.empty((cap, sh.shape[1], 3), dtype=f, device=dev)
        self._pos[:n] = pos
        self._ls[:n] = ls
        self._rot[:n] = rot
        self._op[:n] = op
        self._sh[:n] = sh
        self._count = n

    @property
    def device(self):
        return self._pos.device

    @property
    def sh_coeffs(self) -> int:
        return self._sh.shape[1]

    @classmethod
    def empty(cls, capacity, dtype=np.float32, sh_coeffs=1, device=None):
        z = np.zeros((0, 3), np.float32)
        return cls(z, z, np.zeros((0, 4), np.float32), np.zeros(0, np.float32),
                   np.zeros((0, sh_coeffs, 3), np.float32), capacity, dtype, device)

    def copy(self) -> "Scene3":
        return Scene3(self.positions, self.log_scales, self.rotations, self.opacity_logits,
                      self.sh, self.capacity, device=self.device)

    def to_numpy(self) -> dict:
        """Host copy of the live rows (dict of numpy arrays, plus 'capacity')."""
        return {"positions": self.positions.cpu().numpy(),
                "log_scales": self.log_scales.cpu().numpy(),
                "rotations": self.rotations.cpu().numpy(),
                "opacity_logits": self.opacity_logits.cpu().numpy(),
                "sh": self.sh.cpu().numpy(), "colors": self.colors.cpu().numpy(),
                "capacity": self.capacity}

    @classmethod
    def from_reference(cls, scene, device=None) -> "Scene3":
        """Copy a reference ``splitkit.core.Scene3`` (numpy columns) to the device."""
        return cls(scene.positions, scene.log_scales, scene.rotations, scene.opacity_logits,
                   scene.colors, scene.capacity, device=device)


class Scene2(_DeviceScene):
    """GPU 2-D scene (``splitkit.core.Scene2``, core.py:203-244): float32 SoA columns
    ``positions`` (N,2), ``log_scales`` (N,2), ``thetas`` (N,), ``opacity_logits`` (N,),
    ``colors`` (N,3), pre-reserved at ``capacity`` rows."""

    _columns = ("positions", "log_scales", "thetas", "opacity_logits", "colors")
    _buffers = ("_positions", "_log_scales", "_thetas", "_opacity_logits", "_colors")

    positions = _Column("_positions")
    log_scales = _Column("_log_scales")
    thetas = _Column("_thetas")
    opacity_logits = _Column("_opacity_logits")
    colors = _Column("_colors")

    def __init__(self, positions, log_scales, thetas, opacity_logits, colors, capacity,
                 dtype=np.float32, device=None):
        if capacity < 1:
            raise ValueError("capacity must be positive")
        if np.dtype(dtype) != np.float32:
            raise ValueError("the B200 scene stores float32 columns")
        dev = _dev(device)
        f = torch.float32
        cols = {"positions": _col(positions, 2, f, dev), "log_scales": _col(log_scales, 2, f, dev),
                "thetas": _col(thetas, 0, f, dev), "opacity_logits": _col(opacity_logits, 0, f, dev),
                "colors": _col(colors, 3, f, dev)}
        n = cols["positions"].shape[0]
        for name, col in cols.items():
            if col.shape[0] != n:
                raise ValueError(f"column {name} has length {col.shape[0]} != {n}")
        cap = int(capacity)
        if n > cap:
            raise ValueError(f"count {n} exceeds capacity {cap}")
        self._capacity = cap
        for name, col in cols.items():
            buf = torch.empty((cap,) + tuple(col.shape[1:]), dtype=f, device=dev)
            buf[:n] = col
            setattr(self, "_" + name, buf)
        self._count = n

    @property
    def _cols(self):
        """The reserved buffers by column name (the C-ABI calls take their pointers)."""
        return {name: getattr(self, "_" + name) for name in self._columns}

    @property
    def device(self):
        return self._positions.device

    def copy(self) -> "Scene2":
        return Scene2(self.positions, self.log_scales, self.thetas, self.opacity_logits,
                      self.colors, self.capacity, device=self.device)

    def to_numpy(self) -> dict:
        out = {k: getattr(self, k).cpu().numpy() for k in self._columns}
        out["capacity"] = self.capacity
        return out

    @classmethod
    def from_reference(cls, scene, device=None) -> "Scene2":
        return cls(scene.positions, scene.log_scales, scene.thetas, scene.opacity_logits,
                   scene.colors, scene.capacity, device=device)
