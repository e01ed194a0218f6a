"""Oracle: the ``.igsp`` scene-file layout restated in numpy (TEST INFRASTRUCTURE ONLY).

Restates ``splitkit.io_cli.scene_bytes`` / ``read_scene``
(``/root/reference/pkg/src/splitkit/io_cli.py:32-36,83-134``) on plain dicts of numpy
columns. Errors are reported by the reference exception's class name, so tests can
compare them with the golden vectors (``tests/golden/igsp.npz``, written by the real
reference) and with the GPU loader's exceptions.
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"IGSP"
HEADER = struct.Struct("<4sHBQ")          # io_cli.py:34
RECORD = {2: (("positions", 2), ("log_scales", 2), ("thetas", 0), ("opacity_logits", 0),
              ("colors", 3)),
          3: (("positions", 3), ("log_scales", 3), ("rotations", 4), ("opacity_logits", 0),
              ("colors", 3))}              # io_cli.py:36, column order :71-80


class OracleFormatError(Exception):
    """Carries the reference exception's class name in ``kind``."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def scene_bytes(dims: int, cols: dict) -> bytes:
    """io_cli.py:83-89: header, then every column as little-endian float32, in record order."""
    count = len(cols["positions"])
    out = [HEADER.pack(MAGIC, 1, dims, count)]
    for name, _ in RECORD[dims]:
        out.append(np.ascontiguousarray(cols[name], dtype="<f4").tobytes())
    return b"".join(out)


def read_scene_bytes(data: bytes):
    """io_cli.py:96-134 on an in-memory file: (dims, columns) or OracleFormatError."""
    if data[:4] != MAGIC:
        if len(data) < 4 and MAGIC.startswith(data):
            raise OracleFormatError("SizeMismatchError", "truncated header")
        raise OracleFormatError("BadMagicError", "bad magic")
    if len(data) < HEADER.size:
        raise OracleFormatError("SizeMismatchError", "truncated header")
    _, version, dims, count = HEADER.unpack_from(data)
    if version != 1:
        raise OracleFormatError("UnsupportedVersionError", f"version {version}")
    if dims not in RECORD:
        raise OracleFormatError("SceneFormatError", f"dims {dims}")
    floats = sum(max(w, 1) for _, w in RECORD[dims])
    if len(data) != HEADER.size + count * floats * 4:
        raise OracleFormatError("SizeMismatchError", "payload size")
    cols, off = {}, 0
    for name, w in RECORD[dims]:
        width = max(w, 1)
        flat = np.frombuffer(data, "<f4", count=count * width, offset=HEADER.size + 4 * off * count)
        cols[name] = (flat.reshape(count, w) if w else flat).astype(np.float32)
        off += width
    if dims == 3:
        q = cols["rotations"].astype(np.float64)
        norm = np.sqrt(((q[:, 0] * q[:, 0] + q[:, 1] * q[:, 1]) + q[:, 2] * q[:, 2])
                       + q[:, 3] * q[:, 3])          # np.linalg.norm, summed left to right
        if not np.all(np.isfinite(norm)) or np.any(norm <= 0.0):
            raise OracleFormatError("SceneFormatError", "degenerate quaternion")
        cols["rotations"] = (q / norm[:, None]).astype(np.float32)
    return dims, cols
