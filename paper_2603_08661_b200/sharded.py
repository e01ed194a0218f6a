"""Multi-GPU densification: contiguous Gaussian shards, one process per GPU.

The reference (``splitkit``) is single-process; this module keeps its semantics on a cloud
that is split across ranks in contiguous index ranges ``[lo_r, hi_r)``:

* ``select_candidates_sharded`` is bit-identical to ``select_candidates`` on the
  concatenated statistics (``/root/reference/pkg/src/splitkit/densify_controller.py:80-106``):
  the per-rank radix-select kernels of ``igs_select_shard_*`` with four 256 KB sum
  all-reduces of digit histograms and one 8-byte all-gather of tie counts between them,
  all enqueued on the current stream (no host round trip inside the selection).
* ``las_split_sharded`` splits every rank's masked parents locally.  One all-gather of each
  rank's ``{n_split, flags}`` gives the global budget / domain checks, the batch-global
  quaternion renormalisation rule (``core.py:45-46`` spans the whole masked batch) and
  the global append offsets: the reference layout ``[parents 0..N-1] ++ [children in
  parent order]`` is the concatenation of the ranks' parents followed by the
  concatenation of the ranks' children (``las_split.py:158-179``).
* ``densify_step_sharded`` composes them and returns the reference's ``DensifyEvent``
  with global counts (``densify_controller.py:125-147``).
* ``gather_scene`` all-gathers the compacted rows when every rank needs the whole cloud
  (reported separately: it does not shrink with the number of ranks).

Edge maps shard by view (``shard_range`` over the batch); the median is per view, so that
path has no collective at all.

Collectives go through ``torch.distributed`` on the tensors' device: NCCL over NVLink in
production, gloo in the CPU/one-GPU tests.  The per-rank kernels are pluggable
(``ops=``) only so the protocol can be exercised by CPU tests with a test double; the
product default is the CUDA library, and there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from . import las_split as _las
from .core import Scene3
from .densify_controller import DensifyEvent, DensifyStats, _take_cap
from .schedule import DensifyConfig, is_densify_step, is_warmup_step

ROUNDS = 4  # 16-bit digits of the 64-bit selection key


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
        """(world, *t.shape) stack of every rank's t (same shape on every rank)."""
        if self.world == 1:
            return t.unsqueeze(0).clone()
        parts = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.stack(parts)


# ------------------------------------------------------------------ per-rank CUDA kernels
class CudaSelectShard:
    """The per-rank launches of the sharded radix select (include/igs_b200.h)."""

    def __init__(self, n: int, device):
        self.n = int(n)
        self.device = torch.device(device)
        self.L = _lib.lib()
        nbytes = _lib.query_size(self.L.igs_select_shard_workspace_bytes, self.n)
        self.ws = _lib.workspace(nbytes, self.device, "select_shard")
        self.hist = torch.empty(_lib.IGS_SHARD_HIST_LEN, dtype=torch.int32, device=self.device)
        self.counts = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.local_ties = torch.zeros(1, dtype=torch.int64, device=self.device)

    def keys(self, stats: DensifyStats, cfg: DensifyConfig, step: int) -> torch.Tensor:
        _lib.check(self.L.igs_select_shard_keys(
            stats._grad_sum.data_ptr(), stats._accum_count, stats.edge_score.data_ptr(), self.n,
            float(cfg.grad_threshold), int(is_warmup_step(cfg, step)),
            _lib.IGS_POLICY[cfg.policy], self.hist.data_ptr(), self.ws.data_ptr(),
            self.ws.numel(), _lib.stream_handle()), "select_candidates_sharded")
        return self.hist

    def resolve(self, hist: torch.Tensor, rnd: int, take_cap: int) -> torch.Tensor:
        _lib.check(self.L.igs_select_shard_resolve(
            hist.data_ptr(), rnd, int(take_cap), self.ws.data_ptr(), self.ws.numel(),
            self.counts.data_ptr(), _lib.stream_handle()), "select_candidates_sharded")
        return self.counts

    def digit_hist(self, rnd: int) -> torch.Tensor:
        _lib.check(self.L.igs_select_shard_hist(self.n, rnd, self.hist.data_ptr(),
                                                self.ws.data_ptr(), self.ws.numel(),
                                                _lib.stream_handle()),
                   "select_candidates_sharded")
        return self.hist

    def ties(self) -> torch.Tensor:
        _lib.check(self.L.igs_select_shard_ties(self.n, self.local_ties.data_ptr(),
                                                self.ws.data_ptr(), self.ws.numel(),
                                                _lib.stream_handle()),
                   "select_candidates_sharded")
        return self.local_ties

    def finalize(self, all_ties: torch.Tensor, rank: int) -> torch.Tensor:
        mask = torch.empty(self.n, dtype=torch.uint8, device=self.device)
        all_ties = all_ties.reshape(-1).contiguous()
        _lib.check(self.L.igs_select_shard_finalize(self.n, all_ties.data_ptr(), rank,
                                                    mask.data_ptr(), self.ws.data_ptr(),
                                                    self.ws.numel(), _lib.stream_handle()),
                   "select_candidates_sharded")
        return mask.view(torch.bool)


def select_shard_protocol(ops, stats, cfg, step, take_cap: int, comm: Comm):
    """The collective schedule of the sharded select.  Returns (local bool mask, device
    int64[2] global {#eligible, take}); nothing is read back to the host."""
    hist = comm.all_reduce_sum_(ops.keys(stats, cfg, step))
    counts = ops.resolve(hist, 0, take_cap)
    for rnd in range(1, ROUNDS):
        hist = comm.all_reduce_sum_(ops.digit_hist(rnd))
        ops.resolve(hist, rnd, take_cap)
    all_ties = comm.all_gather(ops.ties())
    return ops.finalize(all_ties, comm.rank), counts


def global_counts(scene, comm: Comm):
    """Every rank's (count, capacity) as a host list, via one small all-gather."""
    t = torch.tensor([scene.count, scene.capacity], dtype=torch.int64, device=_device_of(scene))
    g = comm.all_gather(t).cpu().tolist()
    return [(int(a), int(b)) for a, b in g]


def _device_of(scene):
    return scene.device if hasattr(scene, "device") else torch.device("cpu")


def select_candidates_sharded(stats: DensifyStats, cfg: DensifyConfig, step: int,
                              headroom: int, global_count: int, comm: Comm | None = None,
                              ops=None):
    """Local slice of ``select_candidates(global stats, cfg, step, headroom)``.

    ``headroom`` and ``global_count`` are the GLOBAL scene's (capacity - count) and count;
    take = min(#eligible, headroom, ceil(growth_cap * count - 1e-9)) as at
    densify_controller.py:99-100.  Returns a CUDA bool tensor of this rank's length."""
    comm = comm or Comm()
    if headroom < 0:
        raise ValueError("headroom must be non-negative")
    n = len(stats)
    take_cap = _take_cap(cfg, global_count, headroom) if (headroom > 0 and global_count > 0) else 0
    ops = ops or CudaSelectShard(n, stats._device)
    mask, _ = select_shard_protocol(ops, stats, cfg, step, take_cap, comm)
    return mask


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


def _las_check_global(scene, summaries, caps, c):
    """Host checks of las_split.py:146-155 over all ranks (every rank raises the same
    error).  summaries: per rank (n_split, flags); caps: per rank (count, capacity)."""
    for (ns, _), (cnt, cap) in zip(summaries, caps):
        if cnt + ns > cap:
            raise _las.BudgetError(f"splitting {ns} of {cnt} primitives exceeds shard capacity "
                                   f"{cap}")
    flags = 0
    for ns, fl in summaries:
        if ns:
            flags |= fl
    if flags & _lib.IGS_LAS_BAD_OPACITY:
        raise ValueError("logit requires all values strictly inside (0, 1)")
    if flags & _lib.IGS_LAS_BAD_QUAT:
        raise ValueError("zero or non-finite quaternion")
    return flags


def las_split_sharded(scene: Scene3, mask, c: _las.SplitConstants = _las.SplitConstants(),
                      comm: Comm | None = None, extra=None):
    """Split this rank's masked parents of a contiguous shard in place (las_split.py:158-179
    on the global cloud).  Returns a ShardSplit; ``extra`` (device int64 tensor) rides along
    in the same all-gather (densify_step_sharded uses it for the eligible count)."""
    comm = comm or Comm()
    prep = _las.prepare(scene, mask, c)
    cap = torch.tensor([scene.count, scene.capacity], dtype=torch.int64, device=scene.device)
    parts = [prep.summary, cap] + ([extra] if extra is not None else [])
    g = comm.all_gather(torch.cat(parts)).cpu().tolist()
    summaries = [(int(r[0]), int(r[1])) for r in g]
    caps = [(int(r[2]), int(r[3])) for r in g]
    flags = _las_check_global(scene, summaries, caps, c)
    ns_local = summaries[comm.rank][0]
    if ns_local:
        # apply with this rank's own flags except the batch-global renormalisation bit
        _las.check_and_apply(prep, ns_local, (flags & _lib.IGS_LAS_RENORM), c)
    n_split = [s[0] for s in summaries]
    parents = [cp[0] for cp in caps]
    offset = sum(parents) + sum(n_split[:comm.rank])
    res = ShardSplit(n_split=n_split, parents=parents, flags=flags, offset=offset)
    res.extra = [r[4:] for r in g]
    return res


def densify_step_sharded(scene: Scene3, stats: DensifyStats, cfg: DensifyConfig, step: int,
                         comm: Comm | None = None, caps=None, select_ops=None):
    """One densify event over a sharded cloud (densify_controller.py:125-147 on the global
    scene).  Every rank returns the same DensifyEvent with global counts.  ``caps``: the
    per-rank (count, capacity) list if the caller already has it (else one all-gather)."""
    comm = comm or Comm()
    if not is_densify_step(cfg, step):
        raise ValueError(f"step {step} is not a densify step for this timetable")
    if len(stats) != scene.count:
        raise ValueError("stats length does not match scene count")
    caps = caps or global_counts(scene, comm)
    n_glob = sum(c for c, _ in caps)
    headroom = sum(cap for _, cap in caps) - n_glob
    take_cap = _take_cap(cfg, n_glob, headroom) if (headroom > 0 and n_glob > 0) else 0
    ops = select_ops or CudaSelectShard(len(stats), stats._device)
    mask, counts = select_shard_protocol(ops, stats, cfg, step, take_cap, comm)
    if take_cap > 0:
        res = las_split_sharded(scene, mask, cfg.split_constants, comm, extra=counts)
        eligible = int(res.extra[0][0])
        split = res.total
    else:
        g = counts.cpu().tolist()
        eligible, split = int(g[0]), 0
    stats.reset(scene.count)
    count_after = n_glob + split
    return DensifyEvent(step=step, eligible=eligible, split=split, count_after=count_after)


_FIELDS = (("_pos", 3), ("_ls", 3), ("_rot", 4), ("_op", 1))


def gather_scene(scene: Scene3, parents_before: int, comm: Comm | None = None) -> dict:
    """All-gather the shards into the reference's global layout on every rank: all ranks'
    first ``parents_before`` rows (the parents, split in place), then all ranks' appended
    children, in rank order.  Returns a dict of CUDA tensors (positions, log_scales,
    rotations, opacity_logits, sh).  Rows are packed into one padded float32 block per
    rank for a single all-gather."""
    comm = comm or Comm()
    sh_f = scene._sh.shape[1] * 3
    width = 3 + 3 + 4 + 1 + sh_f
    n = scene.count
    cols = [scene._pos[:n], scene._ls[:n], scene._rot[:n], scene._op[:n, None],
            scene._sh[:n].reshape(n, sh_f)]
    meta = torch.tensor([n, parents_before], dtype=torch.int64, device=scene.device)
    metas = comm.all_gather(meta).cpu().tolist()
    rows = max(m[0] for m in metas)
    block = torch.zeros((rows, width), dtype=torch.float32, device=scene.device)
    block[:n] = torch.cat(cols, dim=1)
    blocks = comm.all_gather(block)
    parents = [blocks[r, :metas[r][1]] for r in range(comm.world)]
    children = [blocks[r, metas[r][1]:metas[r][0]] for r in range(comm.world)]
    full = torch.cat(parents + children)
    out, o = {}, 0
    for name, w in (("positions", 3), ("log_scales", 3), ("rotations", 4),
                    ("opacity_logits", 1), ("sh", sh_f)):
        out[name] = full[:, o:o + w]
        o += w
    out["opacity_logits"] = out["opacity_logits"].reshape(-1)
    out["sh"] = out["sh"].reshape(-1, sh_f // 3, 3)
    return out
