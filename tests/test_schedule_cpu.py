"""Host-side timetable (schedule.py:78-125) against the oracle's restatement, on CPU."""

import pytest

from oracle import select as OS


def test_predicates_match_oracle_over_many_timetables():
    from paper_2603_08661_b200 import DensifyConfig, is_densify_step, is_warmup_step
    for (ws, we, iv, wu) in ((500, 15000, 500, 3), (0, 0, 1, 1), (7, 100, 9, 0), (10, 10, 3, 5),
                             (100, 1000, 250, 2)):
        cfg = DensifyConfig(budget=10, interval=iv, window_start=ws, window_end=we, warmup_steps=wu)
        for step in range(-5, we + 2 * iv + 5):
            assert is_densify_step(cfg, step) == OS.is_densify_step(ws, we, iv, step), step
            assert is_warmup_step(cfg, step) == OS.is_warmup_step(ws, we, iv, wu, step), step
        assert cfg.num_densify_steps == (we - ws) // iv + 1


def test_defaults_and_validation():
    from paper_2603_08661_b200 import DensifyConfig
    cfg = DensifyConfig(budget=1)
    assert (cfg.interval, cfg.window_start, cfg.window_end, cfg.warmup_steps) == (500, 500, 15000, 3)
    assert (cfg.grad_threshold, cfg.growth_cap, cfg.policy) == (0.0002, 0.05, "product")
    assert cfg.num_densify_steps == 30
    for kw in ({"interval": 0}, {"window_start": 10, "window_end": 5}, {"budget": 0},
               {"grad_threshold": -1e-9}, {"policy": "area"}):
        args = dict({"budget": 1}, **kw)
        with pytest.raises(ValueError):
            DensifyConfig(**args)
