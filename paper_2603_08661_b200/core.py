"""Device-resident Gaussian scene for the densification path.

``Scene3`` mirrors ``splitkit.core.Scene3`` (``/root/reference/pkg/src/splitkit/
core.py:122-200``): the same column names (``positions``, ``log_scales``,
``rotations``, ``opacity_logits``, ``colors``), ``count``, ``capacity``,
``validate``, ``copy``, ``empty``.  B200 layout differences:

* storage is pre-reserved at ``capacity`` rows on the GPU (float32 SoA), so a
  split appends children in place instead of re-allocating every column
  (``_append_columns``, core.py:151-157, is an O(N) copy per split);
* spherical harmonics: ``sh`` is a (capacity, K, 3) block whose first
  coefficient triplet IS ``colors`` (K = 1 is the reference's colour-only
  scene, K = 16 is SH degree 3); rows of 48 floats are 16-byte aligned so the
  split clones them with 16-byte vector copies.

Column properties return views of the first ``count`` rows.
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


def _col(x, n_cols, dtype, device):
    t = torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x)
    t = t.to(device=device, dtype=dtype)
    return t.reshape(-1, n_cols) if n_cols else t.reshape(-1)


class Scene3:
    """GPU structure-of-arrays 3D scene with pre-reserved capacity."""

    _columns = ("positions", "log_scales", "rotations", "opacity_logits", "colors")

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
        c = torch.as_tensor(np.asarray(colors) if not isinstance(colors, torch.Tensor) else colors)
        c = c.to(device=dev, dtype=f)
        sh = c if c.ndim == 3 else c.reshape(-1, 1, 3)
        n = pos.shape[0]
        self.capacity = int(capacity)
        for name, col in (("log_scales", ls), ("rotations", rot), ("opacity_logits", op),
                          ("colors", sh)):
            if col.shape[0] != n:
                raise ValueError(f"column {name} has length {col.shape[0]} != {n}")
        if n > self.capacity:
            raise ValueError(f"count {n} exceeds capacity {self.capacity}")
        cap = self.capacity
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

    # -- reference surface ---------------------------------------------------------------
    @property
    def count(self) -> int:
        return self._count

    @property
    def device(self):
        return self._pos.device

    @property
    def sh_coeffs(self) -> int:
        return self._sh.shape[1]

    @property
    def positions(self):
        return self._pos[: self._count]

    @property
    def log_scales(self):
        return self._ls[: self._count]

    @property
    def rotations(self):
        return self._rot[: self._count]

    @property
    def opacity_logits(self):
        return self._op[: self._count]

    @property
    def colors(self):
        """DC colour (count, 3): a strided view of sh[:, 0, :]."""
        return self._sh[: self._count, 0, :]

    @property
    def sh(self):
        return self._sh[: self._count]

    def validate(self):
        if self._count > self.capacity:
            raise ValueError(f"count {self._count} exceeds capacity {self.capacity}")
        return self

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

    # -- growth (used by las_split_batch) ------------------------------------------------
    def _set_count(self, n: int):
        if n > self.capacity:
            raise ValueError(f"count {n} exceeds capacity {self.capacity}")
        self._count = int(n)


class Scene2:
    """GPU 2-D scene (``splitkit.core.Scene2``, core.py:203-244): float32 SoA columns
    ``positions`` (N,2), ``log_scales`` (N,2), ``thetas`` (N,), ``opacity_logits`` (N,),
    ``colors`` (N,3), pre-reserved at ``capacity`` rows."""

    _columns = ("positions", "log_scales", "thetas", "opacity_logits", "colors")

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
        self.capacity = int(capacity)
        if n > self.capacity:
            raise ValueError(f"count {n} exceeds capacity {self.capacity}")
        self._cols = {}
        for name, col in cols.items():
            buf = torch.empty((self.capacity,) + tuple(col.shape[1:]), dtype=f, device=dev)
            buf[:n] = col
            self._cols[name] = buf
        self._count = n

    @property
    def count(self) -> int:
        return self._count

    @property
    def device(self):
        return self._cols["positions"].device

    def __getattr__(self, name):
        cols = self.__dict__.get("_cols")
        if cols is not None and name in cols:
            return cols[name][: self._count]
        raise AttributeError(name)

    def validate(self):
        if self._count > self.capacity:
            raise ValueError(f"count {self._count} exceeds capacity {self.capacity}")
        return self

    def to_numpy(self) -> dict:
        out = {k: getattr(self, k).cpu().numpy() for k in self._columns}
        out["capacity"] = self.capacity
        return out

    @classmethod
    def from_reference(cls, scene, device=None) -> "Scene2":
        return cls(scene.positions, scene.log_scales, scene.thetas, scene.opacity_logits,
                   scene.colors, scene.capacity, device=device)

    def _set_count(self, n: int):
        if n > self.capacity:
            raise ValueError(f"count {n} exceeds capacity {self.capacity}")
        self._count = int(n)
