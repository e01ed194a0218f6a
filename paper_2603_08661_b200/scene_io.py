"""``.igsp`` scene files loaded into and saved from device-resident scenes.

Mirrors ``splitkit.io_cli`` (``/root/reference/pkg/src/splitkit/io_cli.py``):
``scene_bytes`` (:83-89), ``write_scene`` (:92-93), ``read_scene`` (:96-134) and the
``FormatError`` family (:40-57), with the same names, byte layout and exceptions.

Layout (little endian): a 15-byte header ``<4sHBQ`` (magic ``IGSP``, version, dims,
count), then one float32 block per column in the order positions, log_scales, rotations
(quaternions in 3-D, angles in 2-D), opacity_logits, colors.

B200 path: file bytes move in 8 MB pieces through a reusable pool of pinned staging
slots. Worker threads pread / pwrite at the pieces' final offsets (in parallel: the
syscalls release the GIL) and issue each piece's H2D / D2H copy on their own CUDA stream,
straight into / out of the pre-reserved device columns. The rotation block is then
renormalised in place on the GPU (``igs_normalize_quaternions``, bit-identical to the
reference's float64 numpy arithmetic). Writes go to a temp file that is renamed into place.

Extension (version 2): a ``Scene3`` with ``K > 1`` spherical-harmonic triplets per
Gaussian cannot be stored in the reference's 14-float record (:36). It is written as
version 2: the header is followed by ``<H`` K, and the colour block holds (count, K, 3).
Version 1 files are byte-identical to the reference's. The reference reader rejects
version 2 with ``UnsupportedVersionError``.
"""

from __future__ import annotations

import os
import struct
import tempfile

import numpy as np
import torch

from . import _lib
from .core import Scene2, Scene3, _dev

SCENE_MAGIC = b"IGSP"
SCENE_VERSION = 1
SCENE_VERSION_SH = 2
_HEADER = struct.Struct("<4sHBQ")
_SH_FIELD = struct.Struct("<H")
# floats per record: positions + log_scales + rotation + opacity + color (io_cli.py:36)
RECORD_FLOATS = {2: 2 + 2 + 1 + 1 + 3, 3: 3 + 3 + 4 + 1 + 3}


class FormatError(ValueError):
    """Base of the file-format errors (io_cli.py:40-41); a ValueError, as in the reference."""


class SceneFormatError(FormatError):
    """An ``.igsp`` file whose bytes do not follow the layout above (io_cli.py:44-45)."""


class BadMagicError(SceneFormatError):
    """The first four bytes are not ``IGSP``."""


class UnsupportedVersionError(SceneFormatError):
    """A header version this reader does not know."""


class SizeMismatchError(SceneFormatError):
    """File length disagrees with the header's count (or the header itself is cut short)."""


def _columns(scene):
    """(dims, sh_coeffs, [(device tensor, floats per row)]) in file order (io_cli.py:71-80)."""
    if isinstance(scene, Scene3):
        k = scene.sh_coeffs
        colors = scene.colors if k == 1 else scene.sh
        return 3, k, [(scene.positions, 3), (scene.log_scales, 3), (scene.rotations, 4),
                      (scene.opacity_logits, 1), (colors, 3 * k)]
    if isinstance(scene, Scene2):
        return 2, 1, [(scene.positions, 2), (scene.log_scales, 2), (scene.thetas, 1),
                      (scene.opacity_logits, 1), (scene.colors, 3)]
    raise TypeError(f"expected Scene2 or Scene3, got {type(scene).__name__}")


# ---- chunked pinned pipeline ---------------------------------------------------------
# File bytes move in CHUNK-sized pieces through a reusable pool of pinned staging slots:
# worker threads pread / pwrite (the syscalls release the GIL, so page-cache copies run in
# parallel) and issue the H2D / D2H copy of their slot on their own CUDA stream.
CHUNK = 8 << 20
_WORKERS = max(1, min(8, os.cpu_count() or 1))
_POOL = {}


def _slots(device):
    key = (device.index, _WORKERS)
    if key not in _POOL:
        _POOL[key] = [[torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
                      for _ in range(_WORKERS)]
    return _POOL[key]


def _segments(cols, base):
    """[(file offset, device byte view)] for contiguous device columns laid out from `base`."""
    segs, off = [], base
    for t in cols:
        b = t.reshape(-1).view(torch.uint8)
        for a in range(0, b.numel(), CHUNK):
            segs.append((off + a, b[a:a + CHUNK]))
        off += b.numel()
    return segs, off


def _run_chunks(segs, device, fn):
    """Run fn(slot, file_off, dev_bytes, stream) over the segments on the worker pool; the
    caller's stream waits for every worker stream."""
    if not segs:
        return
    import concurrent.futures as cf
    pool = _slots(device)
    nw = min(len(pool), len(segs))
    streams = [torch.cuda.Stream(device) for _ in range(nw)]
    cur = torch.cuda.current_stream(device)
    for st in streams:
        st.wait_stream(cur)

    def work(w):
        events = [None, None]
        with torch.cuda.device(device):
            for i, (off, dev) in enumerate(segs[w::nw]):
                k = i & 1
                if events[k] is not None:
                    events[k].synchronize()
                events[k] = fn(pool[w][k], off, dev, streams[w])
            for e in events:
                if e is not None:
                    e.synchronize()

    with cf.ThreadPoolExecutor(nw) as ex:
        for f in [ex.submit(work, w) for w in range(nw)]:
            f.result()
    for st in streams:
        cur.wait_stream(st)


def _prepare(scene):
    dims, k, cols = _columns(scene)
    scene.validate()
    n = scene.count
    header = _HEADER.pack(SCENE_MAGIC, SCENE_VERSION if k == 1 else SCENE_VERSION_SH, dims, n)
    if k != 1:
        header += _SH_FIELD.pack(k)
    dev_cols = [col.reshape(n, w).contiguous() for col, w in cols]
    segs, end = _segments(dev_cols, len(header))
    return header, segs, end


def _d2h_to(write):
    def fn(slot, off, dev, stream):
        view = slot[:dev.numel()]
        with torch.cuda.stream(stream):
            view.copy_(dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        ev.synchronize()
        write(view, off)
        return None
    return fn


def scene_bytes(scene) -> bytes:
    """The canonical byte string of a scene (io_cli.py:83-89)."""
    header, segs, end = _prepare(scene)
    out = bytearray(end)
    out[:len(header)] = header
    mv = memoryview(out)

    def write(view, off):
        mv[off:off + view.numel()] = view.numpy().data

    _run_chunks(segs, scene.device, _d2h_to(write))
    return bytes(out)


def write_scene(scene, path):
    """Write a scene atomically: temp file in the target directory, then rename (io_cli.py:60-68,92-93).
    Chunks are written with parallel pwrite at their final offsets."""
    header, segs, end = _prepare(scene)
    path = os.fspath(path)
    directory = os.path.dirname(path) or "."
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".tmp.")
    try:
        os.ftruncate(fd, end)
        os.pwrite(fd, header, 0)

        def write(view, off):
            mv = memoryview(view.numpy())
            done = 0
            while done < len(mv):
                done += os.pwrite(fd, mv[done:], off + done)

        _run_chunks(segs, scene.device, _d2h_to(write))
        os.close(fd)
        fd = -1
        os.replace(tmp, path)
    except BaseException:
        if fd >= 0:
            os.close(fd)
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def read_scene(path, capacity=None, device=None):
    """Load a ``Scene2`` / ``Scene3`` onto the GPU, validating the layout and renormalising
    quaternions (io_cli.py:96-134). ``capacity`` (default ``max(count, 1)``, as the
    reference) reserves rows for later splits."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(min(size, _HEADER.size + _SH_FIELD.size))
    if head[:4] != SCENE_MAGIC:
        if len(head) < 4 and SCENE_MAGIC.startswith(head):
            raise SizeMismatchError(f"file too short for a header ({len(head)} bytes)")
        raise BadMagicError(f"not an .igsp file (starts with {head[:4]!r})")
    if len(head) < _HEADER.size:
        raise SizeMismatchError(f"file too short for a header ({len(head)} bytes)")
    _, version, dims, count = _HEADER.unpack_from(head)
    if version not in (SCENE_VERSION, SCENE_VERSION_SH):
        raise UnsupportedVersionError(f".igsp version {version} is not supported")
    if dims not in RECORD_FLOATS:
        raise SceneFormatError(f"scene dimensionality {dims} (expected 2 or 3)")
    hlen, k = _HEADER.size, 1
    if version == SCENE_VERSION_SH:
        if dims != 3 or len(head) < hlen + _SH_FIELD.size:
            raise SceneFormatError("version 2 needs dims 3 and an SH coefficient count")
        (k,) = _SH_FIELD.unpack_from(head, hlen)
        hlen += _SH_FIELD.size
        if k < 1:
            raise SceneFormatError("SH coefficient count must be positive")
    floats = RECORD_FLOATS[dims] + 3 * (k - 1)
    expected = hlen + count * floats * 4
    if size != expected:
        raise SizeMismatchError(f"{size - hlen} payload bytes for {count} records of {floats} "
                                f"floats ({expected - hlen} expected)")
    n = int(count)
    cap = max(n, 1) if capacity is None else int(capacity)
    if cap < n:
        raise ValueError(f"count {n} exceeds capacity {cap}")
    dev = _dev(device)
    if dims == 3:
        scene = Scene3.empty(cap, sh_coeffs=k, device=dev)
        dst = [(scene._pos, 3), (scene._ls, 3), (scene._rot, 4), (scene._op, 1), (scene._sh, 3 * k)]
    else:
        z = np.zeros((0, 2), np.float32)
        scene = Scene2(z, z, np.zeros(0, np.float32), np.zeros(0, np.float32),
                       np.zeros((0, 3), np.float32), cap, device=dev)
        c = scene._cols
        dst = [(c["positions"], 2), (c["log_scales"], 2), (c["thetas"], 1),
               (c["opacity_logits"], 1), (c["colors"], 3)]
    segs, _ = _segments([col.view(cap, w)[:n] for col, w in dst], hlen)
    fd = os.open(path, os.O_RDONLY)
    try:
        def fn(slot, off, devb, stream):
            view = slot[:devb.numel()]
            mv = memoryview(view.numpy())
            got = 0
            while got < len(mv):
                r = os.preadv(fd, [mv[got:]], off + got)
                if r <= 0:
                    raise SizeMismatchError(f"short read at byte {off + got}")
                got += r
            with torch.cuda.stream(stream):
                devb.copy_(view, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            return ev

        _run_chunks(segs, dev, fn)
    finally:
        os.close(fd)
    if dims == 3 and n:
        L = _lib.lib()
        flags = torch.empty(1, dtype=torch.int32, device=dev)
        _lib.check(L.igs_normalize_quaternions(scene._rot.data_ptr(), n, flags.data_ptr(),
                                               _lib.stream_handle(dev)), "read_scene")
        if int(flags.item()):
            raise SceneFormatError("a stored rotation has zero or non-finite norm")
    scene._set_count(n)
    torch.cuda.current_stream(dev).synchronize()
    return scene
