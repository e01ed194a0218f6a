"""Oracle: budgeted split-candidate selection on the CPU (TEST INFRASTRUCTURE ONLY).

Restates ``splitkit.densify_controller`` selection
(``/root/reference/pkg/src/splitkit/densify_controller.py:66-106``) and the
timetable predicates it consults (``schedule.py:116-125``) in numpy.  The
ranking is ``np.argsort(-score, kind="stable")`` over the eligible set, i.e.
the lexicographic order (score descending, index ascending) with +0/-0 tied
and NaN last.
"""

from __future__ import annotations

import math

import numpy as np


def is_densify_step(window_start, window_end, interval, step):
    """schedule.py:116-119."""
    return window_start <= step <= window_end and (step - window_start) % interval == 0


def is_warmup_step(window_start, window_end, interval, warmup_steps, step):
    """schedule.py:122-125."""
    return (is_densify_step(window_start, window_end, interval, step)
            and (step - window_start) // interval < warmup_steps)


def grad_norm(grad_sum, accum_count):
    """densify_controller.py:40-43: running mean, zeros before any accumulation."""
    grad_sum = np.asarray(grad_sum, dtype=np.float64)
    if accum_count == 0:
        return np.zeros_like(grad_sum)
    return grad_sum / accum_count


def take_count(n_eligible, count, headroom, growth_cap):
    """densify_controller.py:99-100 (the 1e-9 slack keeps exact products exact)."""
    cap = math.ceil(growth_cap * count - 1e-9)
    return min(n_eligible, headroom, max(cap, 0))


def select_candidates(grad, edge, warmup, policy, grad_threshold, growth_cap, headroom):
    """densify_controller.py:66-106 with the stats passed as arrays.

    Returns (mask, n_eligible) where n_eligible is what densify_step logs.
    """
    if headroom < 0:
        raise ValueError("headroom must be non-negative")
    grad = np.asarray(grad, dtype=np.float64)
    edge = np.asarray(edge, dtype=np.float64)
    count = len(grad)
    mask = np.zeros(count, dtype=bool)
    eligible_mask = np.ones(count, dtype=bool) if warmup else grad > grad_threshold
    n_eligible = int(eligible_mask.sum())
    if headroom == 0 or count == 0:
        return mask, n_eligible
    eligible = np.flatnonzero(eligible_mask)
    if eligible.size == 0:
        return mask, n_eligible
    take = take_count(eligible.size, count, headroom, growth_cap)
    if take <= 0:
        return mask, n_eligible
    if warmup or policy == "edge":
        score = edge
    elif policy == "grad":
        score = grad
    else:
        score = edge * grad
    order = np.argsort(-score[eligible], kind="stable")
    mask[eligible[order[:take]]] = True
    return mask, n_eligible
