"""CPU test double of the per-rank sharded-select kernels (igs_select_shard_*), so the
collective protocol in paper_2603_08661_b200.sharded can run under gloo on CPU.
TEST INFRASTRUCTURE ONLY: the product path uses sharded.CudaSelectShard."""

from __future__ import annotations

import numpy as np
import torch

from paper_2603_08661_b200.schedule import is_warmup_step

NBINS = 1 << 16
INELIGIBLE = np.uint64(0xFFFFFFFFFFFFFFFF)


def score_keys(score):
    """Order-preserving keys: ascending key == descending score, -0 == +0, NaN last."""
    s = np.where(score == 0.0, 0.0, score).astype(np.float64)
    b = s.view(np.uint64)
    top = np.uint64(1) << np.uint64(63)
    u = np.where((b & top) != 0, ~b, b | top)
    k = ~u
    return np.where(np.isnan(score), np.uint64(0xFFF8000000000000), k)


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
        k = score_keys(sc)
        self.k = np.where(elig, k, INELIGIBLE)
        hist = np.zeros(NBINS + 1, np.int64)
        np.add.at(hist, (self.k[elig] >> np.uint64(48)).astype(np.int64), 1)
        hist[NBINS] = int(elig.sum())
        return torch.from_numpy(hist.astype(np.int32))

    def resolve(self, hist, rnd, take_cap):
        h = hist.cpu().numpy().astype(np.int64)
        if rnd == 0:
            ne = int(h[NBINS])
            self.take = min(ne, take_cap)
            self.counts = torch.tensor([ne, self.take], dtype=torch.int64)
            self.prefix, self.pmask, self.rank = 0, 0, self.take - 1
            self.status = 0 if self.take else 1
        if self.status:
            return self.counts
        cum = np.cumsum(h[:NBINS])
        d = int(np.searchsorted(cum, self.rank, side="right"))
        self.rank -= int(cum[d - 1]) if d else 0
        sh = 48 - 16 * rnd
        self.prefix |= d << sh
        self.pmask |= 0xFFFF << sh
        if rnd == 3:
            self.T = np.uint64(self.prefix)
            self.need = self.rank + 1
        return self.counts

    def digit_hist(self, rnd):
        hist = np.zeros(NBINS + 1, np.int64)
        if not self.status:
            sel = (self.k != INELIGIBLE) & ((self.k & np.uint64(self.pmask)) == np.uint64(self.prefix))
            d = ((self.k[sel] >> np.uint64(48 - 16 * rnd)) & np.uint64(0xFFFF)).astype(np.int64)
            np.add.at(hist, d, 1)
        return torch.from_numpy(hist.astype(np.int32))

    def ties(self):
        c = 0 if self.status else int((self.k == self.T).sum())
        return torch.tensor([c], dtype=torch.int64)

    def finalize(self, all_ties, rank):
        if self.status:
            return torch.zeros(self.n, dtype=torch.bool)
        before = int(all_ties.reshape(-1)[:rank].sum())
        tie = self.k == self.T
        tie_rank = before + np.cumsum(tie) - tie
        m = (self.k < self.T) | (tie & (tie_rank < self.need))
        return torch.from_numpy(m)
