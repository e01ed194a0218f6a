"""Multi-GPU densification: the cloud sharded over ranks, one process per GPU.

The reference (``splitkit``) is single-process; this module keeps its semantics on a cloud
split across ranks.  Every row carries ``gidx``, its index in the global array; selection
ties break by it.  On contiguous shards (``[lo_r, hi_r)`` per rank) a densify event is
exactly the reference's on the global cloud, children included: they get the indices the
reference gives them (all parents first, then every child in parent order,
``las_split.py:158-179``) while staying on their parents' rank.  Capacity is global, as in
the reference: a shard reserves room for the global headroom, so however skewed a selection
is, its children fit on their parents' rank and nothing moves between GPUs.

After an event a rank holds two index ranges (its parents, its children).  The next event is
then exact up to the order it gives children across ranks (rank-major within the event,
where the reference interleaves them by parent index; an exact numbering would need a
segment table that doubles every event).  ``reshard`` restores contiguous shards (one
all-gather of the cloud) so that every event is exact; the tests run event, reshard, event.

* ``densify_step_sharded`` (``densify_controller.py:125-147`` on the global cloud): the
  selection of ``select_candidates`` (``:80-106``, the stable argsort = order by (score key,
  gidx)) and the split, with TWO collectives and ONE host read per event:

  1. ``igs_shard_keys`` -> all-reduce(sum) of a 65536-bin histogram of a monotone digit of the
     score key (256 KB) plus the eligible count;
  2. ``igs_shard_boundary`` (take, boundary digit, this rank's boundary-bucket entries with
     their LAS flags) -> all-gather of the fixed-size records;
  3. ``igs_shard_finalize``: the threshold (key, gidx) by radix select over every rank's
     boundary entries, this rank's mask and its plan (split count, child base, batch flags);
     ``igs_las_split_guarded``; ``igs_shard_child_index``; then the plan is read once.

  A boundary bucket that overflows the record capacity (only for extremely concentrated
  scores) is detected in the plan with nothing written, and steps 2-3 re-run with a record
  sized from the gathered counts.
* ``select_candidates_sharded`` is steps 1-3 without the split (one host read).
* ``las_split_sharded`` splits a caller-given mask: one all-gather of ``{n_split, flags}``
  gives the global budget / domain checks and the batch-global quaternion renormalisation
  rule (``core.py:45-46`` spans the whole masked batch).
* ``gather_scene`` all-gathers the rows and places them by gidx: the reference's layout.

Edge maps shard by view (``shard_range`` over the batch); the median is per view, so that
path has no collective at all.

Collectives go through ``torch.distributed`` on the tensors' device: NCCL in production, gloo
in the CPU / one-GPU tests.  The per-rank kernels are pluggable (``ops=``) only so the
protocol can run in CPU tests with a numpy test double; the product default is the CUDA
library, and there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import las_split as _las
from .densify_controller import DensifyEvent, DensifyStats, _take_cap
from .schedule import DensifyConfig, is_densify_step, is_warmup_step

REC_HDR = 4                  # record header words: #(digit < B), boundary count, their flags, 0
MAX_ENTRIES = 8192           # boundary entries over all ranks that igs_shard_finalize selects
PLAN_WORDS = 16
P_NSPLIT, P_FLAGS, P_STATUS, P_TAKE, P_ELIG, P_CHILD, P_KMINE, P_MAXB = range(8)
P_T, P_G, P_B, P_NEED = 8, 9, 10, 11
STATUS_OK, STATUS_NOTHING, STATUS_OVERFLOW = 0, 1, 2


def shard_range(n: int, rank: int, world: int):
    """Contiguous range [lo, hi) of rank `rank` when n units are split over `world` ranks
    (the first n % world ranks get one extra unit)."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard geometry")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


class Comm:
    """The process group the shards live in (default: the world group; a single process
    without torch.distributed is a world of one)."""

    def __init__(self, group=None):
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0

    def all_reduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """(world, *t.shape) stack of every rank's t (same shape on every rank): one
        all_gather_into_tensor on NCCL, the list form elsewhere (gloo)."""
        if self.world == 1:
            return t.unsqueeze(0)
        t = t.contiguous()
        if dist.get_backend(self.group) == "nccl":
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t, group=self.group)
        return torch.stack(parts)


# ------------------------------------------------------------------ per-rank CUDA kernels
class CudaShardOps:
    """The per-rank launches of the sharded step (include/igs_b200.h igs_shard_*)."""

    def __init__(self, n: int, device):
        self.n = int(n)
        self.device = torch.device(device)
        self.L = _lib.lib()
        nbytes = _lib.query_size(self.L.igs_shard_workspace_bytes, self.n)
        self.ws = _lib.workspace(nbytes, self.device, "shard")
        self.hist = torch.empty(_lib.IGS_SHARD_HIST_LEN + 3, dtype=torch.int32,
                                device=self.device)[:_lib.IGS_SHARD_HIST_LEN]
        self.plan = torch.zeros(PLAN_WORDS, dtype=torch.int64, device=self.device)
        self.mask = torch.empty(self.n, dtype=torch.uint8, device=self.device)
        self.records = {}

    @classmethod
    def cached(cls, owner, n: int, device):
        """One instance per (owner object, n): the buffers are reused event after event."""
        ops = getattr(owner, "_shard_ops", None)
        if ops is None or ops.n != n or ops.device != torch.device(device):
            ops = cls(n, device)
            owner._shard_ops = ops
        return ops

    def keys(self, stats: DensifyStats, cfg: DensifyConfig, step: int) -> torch.Tensor:
        _lib.check(self.L.igs_shard_keys(
            stats._ptr(0), stats._accum_count, stats._ptr(1), self.n,
            float(cfg.grad_threshold), int(is_warmup_step(cfg, step)),
            _lib.IGS_POLICY[cfg.policy], self.hist.data_ptr(), self.ws.data_ptr(),
            self.ws.numel(), _lib.stream_handle()), "densify_step_sharded")
        return self.hist

    def boundary(self, hist, take_cap: int, gidx, scene, beta: float, cap: int):
        rec = self.records.get(cap)
        if rec is None:
            rec = self.records[cap] = torch.empty(REC_HDR + 2 * cap, dtype=torch.int64,
                                                  device=self.device)
        rot, op = _flag_columns(scene)
        _lib.check(self.L.igs_shard_boundary(
            hist.data_ptr(), int(take_cap), gidx.data_ptr(), rot, op, float(beta), self.n,
            int(cap), rec.data_ptr(), self.mask.data_ptr(), self.ws.data_ptr(),
            self.ws.numel(), _lib.stream_handle()), "densify_step_sharded")
        return rec

    def finalize(self, records, rank: int, cap: int, n_global: int, gidx):
        mask = self.mask
        records = records.contiguous()
        _lib.check(self.L.igs_shard_finalize(
            records.data_ptr(), records.shape[0], rank, int(cap), int(n_global),
            gidx.data_ptr(), self.n, mask.data_ptr(), self.plan.data_ptr(), self.ws.data_ptr(),
            self.ws.numel(), _lib.stream_handle()), "densify_step_sharded")
        return mask, self.plan


    def event(self, records, comm, cap: int, n_global: int, gidx, scene, consts, pinned,
              split: bool):
        """finalize -> publish the plan -> (split, child indices) in one library call
        (igs_shard_event); the same launches, in the same order, as the separate calls.  The
        packed arguments are kept per instance; the scene / stream fields are rewritten only
        when a column buffer, the constants or the stream change."""
        a = self.__dict__.get("_ev")
        if a is None:
            a = self._ev = _lib.ShardEventArgs()
            self._ev_addr = ctypes.addressof(a)
            self._ev_key = None
            a.mask, a.plan, a.n = self.mask.data_ptr(), self.plan.data_ptr(), self.n
            a.shard_workspace, a.shard_workspace_bytes = self.ws.data_ptr(), self.ws.numel()
            a.plan_words = PLAN_WORDS
        if split:
            cols = ((scene._pos, scene._ls, scene._rot, scene._op, scene._sh)
                    if hasattr(scene, "_rot") else
                    tuple(scene._cols[k] for k in ("positions", "log_scales", "thetas",
                                                   "opacity_logits", "colors")))
        else:
            cols = ()
        stream = _lib.stream_handle()
        old = self._ev_key
        if (old is None or old[1] != consts or old[2] != stream or old[3] is not pinned
                or len(old[0]) != len(cols) or any(x is not y for x, y in zip(old[0], cols))):
            a.host_plan, a.stream = pinned[0].data_ptr(), stream
            if cols:
                (a.positions, a.log_scales, a.rotations, a.opacity_logits,
                 a.sh_or_colors) = (t.data_ptr() for t in cols)
                a.sh_floats, a.dims = (cols[4].shape[1] * 3, 3) if len(cols[2].shape) == 2 else (3, 2)
                a.alpha, a.log_alpha, a.log_gamma, a.beta = consts
                if self.__dict__.get("_las_ws") is None:  # this shard's own LAS scratch
                    self._las_ws = torch.empty(
                        max(_lib.query_size(self.L.igs_las_workspace_bytes, self.n), 256),
                        dtype=torch.uint8, device=self.device)
                a.las_workspace = self._las_ws.data_ptr()
                a.las_workspace_bytes = self._las_ws.numel()
            self._ev_key = (cols, consts, stream, pinned)
        self._ev_records = records          # alive until the next event on this stream
        a.records, a.world, a.rank = records.data_ptr(), comm.world, comm.rank
        a.record_cap, a.n_global, a.gidx = cap, n_global, gidx.data_ptr()
        a.split = 1 if split else 0
        if split:
            a.reserved_rows = scene.reserved_rows
        rc = self.L.igs_shard_event(self._ev_addr)
        if rc:
            _lib.check(rc, "densify_step_sharded")
        return self.mask, self.plan


def _flag_columns(scene):
    """(rotations or None, opacity_logits) device pointers for the LAS flags of the selected
    parents; no scene (selection only): no flags."""
    if scene is None:
        return None, None
    if hasattr(scene, "_rot"):
        return scene._rot.data_ptr(), scene._op.data_ptr()
    return None, scene._opacity_logits.data_ptr()


def _exchange(ops, stats, cfg, step, take_cap, comm, gidx, scene, beta, cap):
    """The two collective rounds of one event (histogram, boundary records), on the device."""
    hist = comm.all_reduce_sum_(ops.keys(stats, cfg, step))                  # round 1
    rec = ops.boundary(hist, take_cap, gidx, scene, beta, cap)
    return hist, comm.all_gather(rec)                                        # round 2


def _protocol(ops, stats, cfg, step, take_cap, comm, gidx, n_global, scene, beta, cap):
    hist, records = _exchange(ops, stats, cfg, step, take_cap, comm, gidx, scene, beta, cap)
    return hist, ops.finalize(records, comm.rank, cap, n_global, gidx)


def _rerun(ops, hist, take_cap, comm, gidx, n_global, scene, beta, cap):
    rec = ops.boundary(hist, take_cap, gidx, scene, beta, cap)
    return ops.finalize(comm.all_gather(rec), comm.rank, cap, n_global, gidx)


def _publish(plan, pinned):
    """Stream-ordered copy of the plan into pinned memory with a ready word (the host then
    reads it without waiting for the split it guards)."""
    if plan.is_cuda:
        buf, view = pinned
        view[PLAN_WORDS] = -1
        _lib.check(_lib.lib().igs_publish_words(plan.data_ptr(), buf.data_ptr(), PLAN_WORDS,
                                                _lib.stream_handle(plan.device)),
                   "densify_step_sharded")


def _read(plan, pinned):
    if not plan.is_cuda:
        return [int(v) for v in plan.tolist()]
    buf, view = pinned
    _las.wait_word(plan.device, buf, PLAN_WORDS)
    return [int(v) for v in view[:PLAN_WORDS]]


def default_record_cap(world: int) -> int:
    """Boundary entries per rank per record: the kernel's selection capacity split over the
    ranks (a 65536-bin digit leaves ~10^3 scores in the boundary bucket of a 6M cloud)."""
    return max(64, MAX_ENTRIES // max(world, 1))


def _final_large(ops, records, comm, cap, n_global, gidx):
    """The selection for boundary buckets of more than MAX_ENTRIES entries over all ranks (a
    degenerate score distribution, e.g. every warm-up edge score 0): every record holds the
    whole bucket; a stable device sort by (key, gidx) replaces final_kernel's radix select,
    then igs_shard_mask.  Same plan, same result; costs host reads."""
    recs = records.reshape(comm.world, -1)
    plan = ops.plan
    hdr = recs[:, :REC_HDR].cpu().tolist()
    need = int(plan[P_NEED])
    keys, gix, owner = [], [], []
    for r, h in enumerate(hdr):
        m = int(h[1])
        e = recs[r, REC_HDR:REC_HDR + 2 * m].reshape(m, 2)
        keys.append(e[:, 0])
        gix.append(e[:, 1])
        owner.append(torch.full((m,), r, dtype=torch.int64, device=recs.device))
    keys, gix, owner = torch.cat(keys), torch.cat(gix), torch.cat(owner)
    flags_e = gix >> 56
    g = gix & ((1 << 56) - 1)
    signed = keys ^ (-(2 ** 63))             # unsigned order as signed int64
    o = torch.sort(g, stable=True).indices
    o = o[torch.sort(signed[o], stable=True).indices][:need]
    lt = torch.tensor([h[0] for h in hdr], dtype=torch.int64, device=recs.device)
    k_r = lt + torch.bincount(owner[o], minlength=comm.world)
    fl = 0
    for h in hdr:
        fl |= int(h[2])
    for v in flags_e[o].unique().tolist():
        fl |= int(v)
    kr = k_r.cpu().tolist()
    last = o[-1]
    vals = {P_NSPLIT: kr[comm.rank], P_FLAGS: fl, P_STATUS: STATUS_OK, P_KMINE: kr[comm.rank],
            P_CHILD: n_global + sum(kr[:comm.rank]), P_T: int(keys[last]), P_G: int(g[last])}
    for k, v in vals.items():
        plan[k] = v
    _lib.check(ops.L.igs_shard_mask(gidx.data_ptr(), ops.n, plan.data_ptr(), ops.mask.data_ptr(),
                                    ops.ws.data_ptr(), ops.ws.numel(), _lib.stream_handle()),
               "densify_step_sharded")
    return ops.mask, plan


def _resolve_overflow(ops, hist, take_cap, comm, gidx, n_global, scene, beta, maxb):
    """Re-run the boundary round with room for the largest boundary bucket."""
    if maxb * comm.world <= MAX_ENTRIES:
        cap = max(default_record_cap(comm.world), 1 << math.ceil(math.log2(max(maxb, 1))))
        cap = min(cap, MAX_ENTRIES // comm.world)
        return _rerun(ops, hist, take_cap, comm, gidx, n_global, scene, beta, cap)
    rec = ops.boundary(hist, take_cap, gidx, scene, beta, maxb)
    recs = comm.all_gather(rec)
    if hasattr(ops, "final_large"):      # the CPU test double
        return ops.final_large(recs, comm, maxb, n_global, gidx)
    return _final_large(ops, recs, comm, maxb, n_global, gidx)


# ------------------------------------------------------------------ global bookkeeping
def global_counts(scene, comm: Comm):
    """Every rank's (count, capacity) as a host list, via one small all-gather."""
    t = torch.tensor([scene.count, scene.capacity], dtype=torch.int64, device=_device_of(scene))
    g = comm.all_gather(t).cpu().tolist()
    return [(int(a), int(b)) for a, b in g]


def _device_of(scene):
    return scene.device if hasattr(scene, "device") else torch.device("cpu")


@dataclass
class GlobalCloud:
    """The global view a shard keeps: the reference scene's count and capacity."""

    count: int
    capacity: int


def attach(scene, comm: Comm | None = None, caps=None) -> GlobalCloud:
    """Make `scene` this rank's contiguous shard of a global cloud: its global count and
    capacity (sums over the ranks) and each row's global index.  Idempotent; ``caps`` (the
    per-rank (count, capacity) list) saves the all-gather when the caller has it."""
    g = getattr(scene, "_shard_global", None)
    if g is not None:
        return g
    comm = comm or Comm()
    caps = caps or global_counts(scene, comm)
    lo = sum(c for c, _ in caps[:comm.rank])
    gidx = torch.empty(scene.reserved_rows, dtype=torch.int64, device=scene.device)
    gidx[:scene.count] = torch.arange(lo, lo + scene.count, device=scene.device)
    scene._gidx = gidx
    scene._shard_global = GlobalCloud(sum(c for c, _ in caps), sum(cp for _, cp in caps))
    return scene._shard_global


def reshard(scene, comm: Comm | None = None):
    """Re-cut the cloud into contiguous shards of the reference's global array (one all-gather
    of every row, then each rank keeps its range): afterwards gidx = lo_r + local index and
    the next densify event is exactly the reference's.  Returns (lo, hi)."""
    comm = comm or Comm()
    glob = attach(scene, comm)
    full = gather_scene(scene, comm=comm)
    n = full["positions"].shape[0]
    lo, hi = shard_range(n, comm.rank, comm.world)
    k = hi - lo
    _reserve(scene, k)
    scene._pos[:k] = full["positions"][lo:hi]
    scene._ls[:k] = full["log_scales"][lo:hi]
    scene._rot[:k] = full["rotations"][lo:hi]
    scene._op[:k] = full["opacity_logits"][lo:hi]
    scene._sh[:k] = full["sh"][lo:hi]
    scene._capacity = max(scene._capacity, k)
    scene._set_count(k)
    scene._gidx[:k] = torch.arange(lo, hi, dtype=torch.int64, device=scene.device)
    glob.count = n
    return lo, hi


def detach(scene):
    """Forget the shard's global view (the next step re-attaches it as a contiguous shard)."""
    scene.__dict__.pop("_shard_global", None)
    scene.__dict__.pop("_gidx", None)


def _reserve(scene, rows: int):
    """Physical rows for this shard (a shard holds the global headroom's worth of children at
    most): grow the columns and the global-index column together."""
    if scene.reserved_rows < rows:
        scene._reserve(rows)
    if scene._gidx.shape[0] < scene.reserved_rows:
        g = torch.empty(scene.reserved_rows, dtype=torch.int64, device=scene.device)
        g[:scene.count] = scene._gidx[:scene.count]
        scene._gidx = g


def _take_cap_global(cfg, glob: GlobalCloud) -> int:
    headroom = glob.capacity - glob.count
    return _take_cap(cfg, glob.count, headroom) if (headroom > 0 and glob.count > 0) else 0


# ------------------------------------------------------------------ public API
def select_candidates_sharded(stats: DensifyStats, cfg: DensifyConfig, step: int,
                              headroom: int, global_count: int, comm: Comm | None = None,
                              ops=None, gidx=None, scene=None, record_cap=None,
                              return_plan=False):
    """This rank's slice of ``select_candidates(global stats, cfg, step, headroom)``
    (densify_controller.py:80-106).  ``headroom`` / ``global_count`` are the global scene's;
    ``gidx`` the rows' global indices (default: a contiguous shard).  Returns a bool tensor
    of this rank's length (and the plan words when ``return_plan``)."""
    comm = comm or Comm()
    if headroom < 0:
        raise ValueError("headroom must be non-negative")
    n = len(stats)
    dev = stats._device
    take_cap = _take_cap(cfg, global_count, headroom) if (headroom > 0 and global_count > 0) else 0
    if gidx is None:
        sizes = comm.all_gather(torch.tensor([n], dtype=torch.int64, device=dev)).cpu()
        lo = int(sizes[:comm.rank].sum())
        gidx = torch.arange(lo, lo + n, dtype=torch.int64, device=dev)
    ops = ops or CudaShardOps(n, dev)
    beta = cfg.split_constants.device_constants()[3]
    cap = record_cap or default_record_cap(comm.world)
    hist, (mask, plan) = _protocol(ops, stats, cfg, step, take_cap, comm, gidx, global_count,
                                   scene, beta, cap)
    pinned = _las.pinned_summary(dev, PLAN_WORDS + 1) if dev.type == "cuda" else None
    _publish(plan, pinned)
    p = _read(plan, pinned)
    while p[P_STATUS] == STATUS_OVERFLOW:
        mask, plan = _resolve_overflow(ops, hist, take_cap, comm, gidx, global_count, scene, beta,
                                       p[P_MAXB])
        _publish(plan, pinned)
        p = _read(plan, pinned)
    return (mask.view(torch.bool), p) if return_plan else mask.view(torch.bool)


def densify_step_sharded(scene, stats: DensifyStats, cfg: DensifyConfig, step: int,
                         comm: Comm | None = None, caps=None, select_ops=None) -> DensifyEvent:
    """One densify event on this rank's shard (densify_controller.py:125-147 on the global
    scene).  Every rank returns the same DensifyEvent with global counts.  ``caps``: the
    per-rank (count, capacity) list for the first call (else one all-gather)."""
    comm = comm or Comm()
    if not is_densify_step(cfg, step):
        raise ValueError(f"step {step} is not a densify step for this timetable")
    if len(stats) != scene.count:
        raise ValueError("stats length does not match scene count")
    glob = attach(scene, comm, caps)
    take_cap = _take_cap_global(cfg, glob)
    n = scene.count
    _reserve(scene, n + min(take_cap, n))
    ops = select_ops or CudaShardOps.cached(scene, n, stats._device)
    c = cfg.split_constants
    alpha, log_alpha, log_gamma, beta = c.device_constants()
    gidx = scene._gidx
    cap = default_record_cap(comm.world)
    pinned = ops.__dict__.get("_pinned")
    if pinned is None:
        pinned = ops._pinned = _las.pinned_summary(scene.device, PLAN_WORDS + 1)
    if isinstance(ops, CudaShardOps):   # finalize, publish, split, child indices: one call
        hist = comm.all_reduce_sum_(ops.keys(stats, cfg, step))             # round 1
        rec = ops.boundary(hist, take_cap, gidx, scene, beta, cap)
        records = comm.all_gather(rec).contiguous() if comm.world > 1 else rec  # round 2
        mask, plan = ops.event(records, comm, cap, glob.count, gidx, scene,
                               (alpha, log_alpha, log_gamma, beta), pinned, take_cap > 0)
    else:
        hist, records = _exchange(ops, stats, cfg, step, take_cap, comm, gidx, scene, beta,
                                  cap)
        mask, plan = ops.finalize(records, comm.rank, cap, glob.count, gidx)
        _launch_split(scene, mask, plan, pinned, take_cap, gidx, n, alpha, log_alpha, log_gamma,
                      beta)
    while True:
        p = _read(plan, pinned)  # the event's one host read (the split may still be running)
        if p[P_STATUS] != STATUS_OVERFLOW:
            break
        mask, plan = _resolve_overflow(ops, hist, take_cap, comm, gidx, glob.count, scene,
                                       beta, p[P_MAXB])            # nothing was written
        _launch_split(scene, mask, plan, pinned, take_cap, gidx, n, alpha, log_alpha, log_gamma,
                      beta)
    split = p[P_TAKE] if p[P_STATUS] == STATUS_OK else 0
    if split and p[P_FLAGS] & _lib.IGS_LAS_BAD_OPACITY:
        raise ValueError("logit requires all values strictly inside (0, 1)")
    if split and p[P_FLAGS] & _lib.IGS_LAS_BAD_QUAT:
        raise ValueError("zero or non-finite quaternion")
    if split:
        if n + p[P_KMINE] > scene._capacity:   # this shard's share of the global headroom
            scene._capacity = scene.reserved_rows
        scene._set_count(n + p[P_KMINE])
    glob.count += split
    stats.reset(scene.count)
    return DensifyEvent(step=step, eligible=p[P_ELIG], split=split, count_after=glob.count)


def _launch_split(scene, mask, plan, pinned, take_cap, gidx, n, alpha, log_alpha, log_gamma,
                  beta):
    """publish the plan, then the guarded split and the children's global indices."""
    _publish(plan, pinned)
    if take_cap > 0:
        _split_guarded(scene, mask, plan, alpha, log_alpha, log_gamma, beta)
        _lib.check(_lib.lib().igs_shard_child_index(gidx.data_ptr(), n, plan.data_ptr(),
                                                    _lib.stream_handle()),
                   "densify_step_sharded")


def _split_guarded(scene, mask, guard, alpha, log_alpha, log_gamma, beta):
    L = _lib.lib()
    n = scene.count
    ws = _lib.workspace(_lib.query_size(L.igs_las_workspace_bytes, n), scene.device, "las")
    if hasattr(scene, "_rot"):
        args = (scene._pos.data_ptr(), scene._ls.data_ptr(), scene._rot.data_ptr(),
                scene._op.data_ptr(), scene._sh.data_ptr(), scene._sh.shape[1] * 3, 3)
    else:
        cols = scene._cols
        args = (cols["positions"].data_ptr(), cols["log_scales"].data_ptr(),
                cols["thetas"].data_ptr(), cols["opacity_logits"].data_ptr(),
                cols["colors"].data_ptr(), 3, 2)
    _lib.check(L.igs_las_split_guarded(*args, n, scene.reserved_rows, mask.data_ptr(), alpha,
                                       log_alpha, log_gamma, beta, guard.data_ptr(),
                                       ws.data_ptr(), ws.numel(), _lib.stream_handle()),
               "densify_step_sharded")


@dataclass
class ShardSplit:
    """Outcome of one sharded split on this rank."""

    n_split: list          # per rank
    parents: list          # per rank, count before the split
    flags: int             # OR over ranks of the igs_las_flags
    offset: int            # global index of this rank's first appended child

    @property
    def total(self):
        return sum(self.n_split)


def _las_check_global(summaries, count: int, capacity: int):
    """The reference's checks (las_split.py:146-155) on the GLOBAL scene: one count and one
    capacity (sums over the ranks), the domain flags of every rank's masked parents.
    summaries: per rank (n_split, flags).  Every rank raises the same error."""
    total = sum(ns for ns, _ in summaries)
    if count + total > capacity:
        raise _las.BudgetError(f"splitting {total} of {count} primitives exceeds capacity "
                               f"{capacity}")
    flags = 0
    for ns, fl in summaries:
        if ns:
            flags |= fl
    if total and flags & _lib.IGS_LAS_BAD_OPACITY:
        raise ValueError("logit requires all values strictly inside (0, 1)")
    if total and flags & _lib.IGS_LAS_BAD_QUAT:
        raise ValueError("zero or non-finite quaternion")
    return flags


def las_split_sharded(scene, mask, c: _las.SplitConstants = _las.SplitConstants(),
                      comm: Comm | None = None):
    """Split this rank's masked parents in place (las_split.py:158-179 on the global cloud):
    one all-gather of {n_split, flags, count, capacity}; children keep to their parents' rank
    and get the global indices the reference gives them."""
    comm = comm or Comm()
    glob = attach(scene, comm)
    n = scene.count
    prep = _las.prepare(scene, mask, c)
    caps_now = torch.tensor([scene.count, scene.capacity], dtype=torch.int64, device=scene.device)
    g = comm.all_gather(torch.cat([prep.summary, caps_now])).cpu().tolist()
    summaries = [(int(r[0]), int(r[1])) for r in g]
    caps = [(int(r[2]), int(r[3])) for r in g]
    flags = _las_check_global(summaries, glob.count, glob.capacity)
    ns_local = summaries[comm.rank][0]
    n_split = [s[0] for s in summaries]
    offset = glob.count + sum(n_split[:comm.rank])
    if ns_local:
        _reserve(scene, n + ns_local)           # the shard's share of the global headroom
        scene._capacity = max(scene._capacity, n + ns_local)
        _las.check_and_apply(prep, ns_local, flags & _lib.IGS_LAS_RENORM, c)
        plan = torch.tensor([0, 0, STATUS_OK, 0, 0, offset, ns_local, 0] + [0] * 8,
                            dtype=torch.int64, device=scene.device)
        _lib.check(_lib.lib().igs_shard_child_index(scene._gidx.data_ptr(), n, plan.data_ptr(),
                                                    _lib.stream_handle()), "las_split_sharded")
    glob.count += sum(n_split)
    return ShardSplit(n_split=n_split, parents=[cp[0] for cp in caps], flags=flags,
                      offset=offset)


_FIELDS = ("positions", "log_scales", "rotations", "opacity_logits", "sh")


def gather_scene(scene, parents_before: int | None = None, comm: Comm | None = None) -> dict:
    """All-gather the shards into the reference's global layout on every rank: each row at
    its global index.  Returns a dict of tensors (positions, log_scales, rotations,
    opacity_logits, sh).  (``parents_before`` is accepted for compatibility; the global
    indices carry the layout.)"""
    comm = comm or Comm()
    sh_f = scene._sh.shape[1] * 3
    width = 3 + 3 + 4 + 1 + sh_f
    n = scene.count
    gidx = getattr(scene, "_gidx", None)
    if gidx is None:  # a plain contiguous shard
        sizes = comm.all_gather(torch.tensor([n], dtype=torch.int64, device=scene.device)).cpu()
        lo = int(sizes[:comm.rank].sum())
        gidx = torch.arange(lo, lo + n, dtype=torch.int64, device=scene.device)
    cols = [scene._pos[:n], scene._ls[:n], scene._rot[:n], scene._op[:n, None],
            scene._sh[:n].reshape(n, sh_f)]
    counts = comm.all_gather(torch.tensor([n], dtype=torch.int64, device=scene.device))
    counts = counts.reshape(-1).cpu().tolist()
    rows = max(counts)
    block = torch.zeros((rows, width + 2), dtype=torch.float32, device=scene.device)
    block[:n, :width] = torch.cat(cols, dim=1)
    block[:n, width:] = gidx[:n].to(torch.int64).view(torch.int32).reshape(n, 2).view(
        torch.float32)
    blocks = comm.all_gather(block)
    total = sum(counts)
    full = torch.empty((total, width), dtype=torch.float32, device=scene.device)
    for r in range(comm.world):
        b = blocks[r, :counts[r]]
        idx = b[:, width:].contiguous().view(torch.int32).view(torch.int64).reshape(-1)
        full[idx] = b[:, :width]
    out, o = {}, 0
    for name, w in zip(_FIELDS, (3, 3, 4, 1, sh_f)):
        out[name] = full[:, o:o + w]
        o += w
    out["opacity_logits"] = out["opacity_logits"].reshape(-1)
    out["sh"] = out["sh"].reshape(-1, sh_f // 3, 3)
    return out
