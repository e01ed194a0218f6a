"""CPU test double of the per-rank sharded-step kernels (igs_shard_keys / _boundary /
_finalize), so the collective protocol in paper_2603_08661_b200.sharded can run under gloo
on CPU.  It restates the kernels' arithmetic in numpy (same digit, same records, same plan).
TEST INFRASTRUCTURE ONLY: the product path uses sharded.CudaShardOps."""

from __future__ import annotations

import numpy as np
import torch

from paper_2603_08661_b200 import sharded as S
from paper_2603_08661_b200.schedule import is_warmup_step

NBINS = 1 << 16
INELIGIBLE = np.uint64(0xFFFFFFFFFFFFFFFF)
NAN_KEY = np.uint64(0xFFF8000000000000)
T_LO, T_HI = 984064, 984064 + 65532


def score_keys(score):
    """Order-preserving keys: ascending key == descending score, -0 == +0, NaN last."""
    s = np.where(score == 0.0, 0.0, score).astype(np.float64)
    b = s.view(np.uint64)
    top = np.uint64(1) << np.uint64(63)
    u = np.where((b & top) != 0, ~b, b | top)
    k = ~u
    return np.where(np.isnan(score), NAN_KEY, k)


def key_digit(k):
    """select_shard.cu key_digit, vectorised."""
    u = ~k
    pos = (u >> np.uint64(63)) != 0
    b = u & np.uint64(0x7FFFFFFFFFFFFFFF)
    t = np.clip((b >> np.uint64(42)).astype(np.int64), T_LO, T_HI)
    d = np.where(pos & (b != 0), 1 + (T_HI - t), 65534)
    return np.where(k == NAN_KEY, 65535, d).astype(np.int64)


class NumpyShardOps:
    def __init__(self, n):
        self.n = n

    def keys(self, stats, cfg, step):
        g = stats.grad_norm.cpu().numpy()
        e = stats.edge_score.cpu().numpy()
        warm = is_warmup_step(cfg, step)
        elig = np.ones(self.n, bool) if warm else g > cfg.grad_threshold
        if warm or cfg.policy == "edge":
            sc = e
        elif cfg.policy == "grad":
            sc = g
        else:
            sc = e * g
        self.k = np.where(elig, score_keys(sc), INELIGIBLE)
        self.elig = elig
        hist = np.zeros(NBINS + 1, np.int64)
        np.add.at(hist, key_digit(self.k[elig]), 1)
        hist[NBINS] = int(elig.sum())
        return torch.from_numpy(hist.astype(np.int32))

    def boundary(self, hist, take_cap, gidx, scene, beta, cap):
        h = hist.cpu().numpy().astype(np.int64)
        ne = int(h[NBINS])
        self.take = min(ne, int(take_cap))
        self.n_elig = ne
        self.B, self.need = NBINS, 0
        if self.take:
            cum = np.cumsum(h[:NBINS])
            self.B = int(np.searchsorted(cum, self.take - 1, side="right"))
            self.need = self.take - (int(cum[self.B - 1]) if self.B else 0)
        rec = np.zeros(S.REC_HDR + 2 * cap, np.int64)
        if self.take:
            d = key_digit(self.k)
            gi = gidx.cpu().numpy()
            rec[0] = int((self.elig & (d < self.B)).sum())
            sel = np.flatnonzero(self.elig & (d == self.B))
            rec[1] = len(sel)
            m = min(len(sel), cap)
            rec[S.REC_HDR:S.REC_HDR + 2 * m:2] = self.k[sel[:m]].view(np.int64)
            rec[S.REC_HDR + 1:S.REC_HDR + 2 * m:2] = gi[sel[:m]]
        return torch.from_numpy(rec)

    def final_large(self, records, comm, cap, n_global, gidx):
        return self.finalize(records, comm.rank, cap, n_global, gidx)

    def finalize(self, records, rank, cap, n_global, gidx):
        recs = records.cpu().numpy().reshape(records.shape[0], -1)
        plan = np.zeros(S.PLAN_WORDS, np.int64)
        plan[S.P_TAKE], plan[S.P_ELIG] = self.take, self.n_elig
        plan[S.P_MAXB] = int(recs[:, 1].max())
        mask = np.zeros(self.n, bool)
        if not self.take:
            plan[S.P_STATUS] = S.STATUS_NOTHING
        elif (recs[:, 1] > cap).any():
            plan[S.P_STATUS] = S.STATUS_OVERFLOW
        else:
            keys, gix, owner = [], [], []
            for r, rec in enumerate(recs):
                m = int(rec[1])
                keys.append(rec[S.REC_HDR:S.REC_HDR + 2 * m:2].view(np.uint64))
                gix.append(rec[S.REC_HDR + 1:S.REC_HDR + 2 * m:2] & ((1 << 56) - 1))
                owner.append(np.full(m, r))
            keys, gix, owner = map(np.concatenate, (keys, gix, owner))
            order = np.lexsort((gix, keys))[:self.need]
            T, G = keys[order[-1]], gix[order[-1]]
            k_r = recs[:, 0] + np.bincount(owner[order], minlength=len(recs))
            plan[S.P_NSPLIT] = plan[S.P_KMINE] = k_r[rank]
            plan[S.P_CHILD] = n_global + int(k_r[:rank].sum())
            d = key_digit(self.k)
            gi = gidx.cpu().numpy()
            mask = self.elig & ((d < self.B) | ((d == self.B) & (
                (self.k < T) | ((self.k == T) & (gi <= G)))))
        return torch.from_numpy(mask.astype(np.uint8)), torch.from_numpy(plan)
