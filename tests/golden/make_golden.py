"""Generate golden vectors by running the REAL reference (``splitkit``) in the build container.

Usage (build container only -- ``/root/reference`` does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/{edge,nms,median,las,select,sample,las2d,igsp,splat2d,cli}.npz``
(``make_golden.py NAME ...`` regenerates only those).  The fixtures are
small (<= 128x128 images, <= 2k Gaussians) and committed; tests compare the
oracle against them on CPU and the CUDA path against them on the GPU.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from splitkit.core import Scene2, Scene3  # noqa: E402
from splitkit.densify_controller import (DensifyStats, accumulate_grads,  # noqa: E402
                                         densify_step, select_candidates)
from splitkit.io_cli import read_scene, scene_bytes  # noqa: E402
from splitkit.edge_pipeline import (GradientField, gaussian_blur_5x5,  # noqa: E402
                                    importance_pipeline, median_normalize,
                                    nms_thin, sample_scores, sobel_gradients,
                                    to_grayscale)
from splitkit.las_split import (BudgetError, SplitConstants, las_split_batch,  # noqa: E402
                                las_split_batch_2d)
from splitkit.schedule import DensifyConfig  # noqa: E402


def synth_view(h, w, seed):
    """SURVEY.md section 8(d) view generator at an arbitrary size (8-bit quantised)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w]
    out = np.empty((h, w, 3))
    for c in range(3):
        ph = rng.uniform(0, 2 * np.pi)
        out[..., c] = 0.5 + 0.5 * np.sin(xx / 37 + ph) * np.cos(yy / 53 - ph)
    out += rng.normal(0, 0.05, out.shape)
    return np.floor(np.clip(out, 0, 1) * 255 + 0.5) / 255


def edge_cases():
    rng = np.random.default_rng(2024)
    cases = {}
    # reference conftest square target (pkg/tests/conftest.py:5-13)
    yy, xx = np.mgrid[0:64, 0:64]
    sq = np.zeros((64, 64, 3))
    sq[..., 0] = xx / 63 * 0.4
    sq[..., 1] = 0.15
    sq[..., 2] = yy / 63 * 0.4
    sq[16:38, 12:34] = 1.0
    cases["square_target"] = (sq, 1.0)
    # acceptance criterion 4 square (test_acceptance.py:184-201) and step edge
    a = np.zeros((128, 128, 3))
    a[32:76, 24:68] = 1.0
    cases["square128"] = (a, 1.0)
    step = np.full((128, 128), 0.2)
    step[:, 64:] = 0.8
    cases["step128_gray"] = (step, 1.0)
    hstep = np.full((40, 56), 0.2)
    hstep[20:, :] = 0.8
    cases["hstep_gray"] = (hstep, 1.0)
    cases["rand16"] = (np.random.default_rng(12).random((16, 16, 3)), 1.0)
    cases["gray12"] = (np.random.default_rng(13).random((12, 12)), 1.0)
    cases["synth"] = (synth_view(97, 131, 1000), 1.0)
    blocks = np.kron(rng.integers(0, 256, (7, 9, 3)), np.ones((16, 16, 1)))[:100, :129] / 255.0
    cases["blocks16"] = (blocks, 1.0)
    rect = np.zeros((77, 101, 3))
    rect[20:50, 30:80] = 1.0
    cases["white_rect"] = (rect, 1.0)
    cases["uniform"] = (rng.random((64, 80, 3)), 1.0)
    cases["uniform_f32"] = (rng.random((33, 47, 3)).astype(np.float32), 1.0)
    cases["tiny3x3"] = (rng.random((3, 3, 3)), 1.0)
    cases["tiny3x7"] = (rng.random((3, 7, 3)), 1.0)
    cases["tall70x3"] = (rng.random((70, 3, 3)), 1.0)
    cases["flat"] = (np.zeros((16, 16, 3)), 1.0)
    cases["white"] = (np.ones((20, 24, 3)), 1.0)
    cases["gray_wide"] = (rng.normal(0, 3.0, (48, 52)), 1.0)  # gray input: not clipped
    cases["rgb_outside"] = (rng.normal(0.5, 0.6, (40, 44, 3)), 1.0)  # gray clip active
    g = rng.random((45, 61))
    for s in (0.3, 0.5, 0.7, 2.2, 3.0):
        cases[f"sigma{s}"] = (g, s)
    # non-finite pixels (their own generator, so the cases above keep their draws)
    nf = np.floor(np.random.default_rng(77).random((40, 52, 3)) * 255) / 255
    nf[10, 10, 0] = np.nan
    nf[25, 30, 2] = np.inf
    nf[33, 5, 1] = -np.inf
    cases["nonfinite"] = (nf, 1.0)
    out = {}
    for name, (img, sigma) in cases.items():
        gray = img if img.ndim == 2 else to_grayscale(img)
        blurred = gaussian_blur_5x5(gray, sigma)
        field = sobel_gradients(blurred)
        thinned = nms_thin(field)
        out[f"{name}/image"] = img
        out[f"{name}/sigma"] = np.float64(sigma)
        out[f"{name}/gray"] = np.asarray(gray, dtype=np.float64)
        out[f"{name}/blurred"] = blurred
        out[f"{name}/magnitude"] = field.magnitude
        out[f"{name}/orientation"] = field.orientation
        out[f"{name}/thinned"] = thinned
        out[f"{name}/importance"] = importance_pipeline(img, sigma)
        assert np.array_equal(out[f"{name}/importance"], median_normalize(thinned))
    return out


def nms_cases():
    out = {}
    rng = np.random.default_rng(7)  # test_edge_pipeline.py:188-194
    for i in range(20):
        mag = rng.random((12, 13))
        ori = rng.random((12, 13)) * np.pi
        out[f"rand{i}/mag"], out[f"rand{i}/ori"] = mag, ori
        out[f"rand{i}/out"] = nms_thin(GradientField(mag, ori))
    mag = np.zeros((3, 5))
    mag[1, 1:4] = 0.7
    ori = np.zeros((3, 5))
    out["plateau/mag"], out["plateau/ori"] = mag, ori
    out["plateau/out"] = nms_thin(GradientField(mag, ori))
    # exact bin boundaries and ties
    rng = np.random.default_rng(77)
    mag = np.round(rng.random((31, 29)) * 4) / 4
    ori = rng.choice(np.array([0.0, np.pi / 8, np.pi / 4, 3 * np.pi / 8, np.pi / 2,
                               5 * np.pi / 8, 3 * np.pi / 4, 7 * np.pi / 8,
                               np.nextafter(np.pi, 0)]), size=(31, 29))
    out["ties/mag"], out["ties/ori"] = mag, ori
    out["ties/out"] = nms_thin(GradientField(mag, ori))
    return out


def median_cases():
    out = {}
    rng = np.random.default_rng(10)
    arrays = {
        "rand8x8": rng.random((8, 8)) * (rng.random((8, 8)) > 0.5),
        "odd": np.array([0.0, 3.0, 1.0, 2.0, 0.0]),
        "even": np.array([0.0, 4.0, 1.0, 2.0, 3.0]),
        "zeros": np.zeros((5, 5)),
        "neg_mixed": rng.normal(size=(17, 19)),
        "ties": np.round(rng.random((40, 40)) * 3) / 3,
        "spread": np.exp(rng.uniform(-80, 5, (64, 70))) * (rng.random((64, 70)) > 0.6),
        "one": np.array([[0.0, 0.25], [0.0, 0.0]]),
        "clamp": np.array([1.0] * 8 + [10.0]),
    }
    for name, a in arrays.items():
        out[f"{name}/in"] = a
        out[f"{name}/out"] = median_normalize(a)
    return out


def random_scene(rng, n, capacity, offnorm=0):
    """test_acceptance.py:50-58 generator (+ optional off-norm quaternions)."""
    positions = rng.normal(0.0, 1.0, (n, 3))
    log_scales = rng.uniform(-0.7, 0.7, (n, 3))
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    if offnorm:
        quats[rng.choice(n, size=min(offnorm, n), replace=False)] *= 1.01
    opacity = rng.normal(0.0, 1.5, n)
    colors = rng.random((n, 3))
    return Scene3(positions, log_scales, quats, opacity, colors, capacity=capacity)


def las_cases():
    out = {}
    rng = np.random.default_rng(303)
    specs = [("c%d" % i, int(rng.integers(1, 65)), 0.4, 0) for i in range(30)]
    specs += [("allmask2k", 2000, 1.0, 0), ("sparse2k", 2000, 0.05, 0),
              ("offnorm", 500, 0.5, 3), ("empty", 50, 0.0, 0), ("single", 1, 1.0, 0)]
    for name, n, p, off in specs:
        scene = random_scene(rng, n, 2 * n + 1, off)
        if name == "offnorm":
            ls = scene.log_scales
            ls[:20, 1] = ls[:20, 0]          # argmax ties -> lowest index
            ls[20:40] = ls[20:40, :1]
        mask = rng.random(n) < p
        if name == "offnorm":
            mask[:60] = True
        before = scene.copy()
        las_split_batch(scene, mask, SplitConstants())
        for col in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
            out[f"{name}/in_{col}"] = getattr(before, col)
            out[f"{name}/out_{col}"] = getattr(scene, col)
        out[f"{name}/mask"] = mask
        out[f"{name}/capacity"] = np.int64(before.capacity)
    # non-default constants
    scene = random_scene(rng, 300, 700)
    mask = rng.random(300) < 0.5
    before = scene.copy()
    consts = SplitConstants(alpha=0.3, gamma_axis=1.0, beta=0.9)
    las_split_batch(scene, mask, consts)
    for col in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
        out[f"consts/in_{col}"] = getattr(before, col)
        out[f"consts/out_{col}"] = getattr(scene, col)
    out["consts/mask"] = mask
    out["consts/capacity"] = np.int64(700)
    out["consts/constants"] = np.array([0.3, 1.0, 0.9])
    # non-finite log-scales / positions on masked parents (np.argmax takes the first NaN; exp
    # of +-inf), from their own generator so the cases above keep their draws
    r2 = np.random.default_rng(909)
    scene = random_scene(r2, 64, 129)
    ls = scene.log_scales
    ls[0, 1] = np.nan
    ls[1, :] = np.nan
    ls[2, 2] = np.inf
    ls[3, 0] = -np.inf
    ls[4, :] = -np.inf
    scene.positions[5, 0] = np.nan
    scene.positions[6, 2] = np.inf
    mask = np.ones(64, dtype=bool)
    mask[7] = False
    before = scene.copy()
    with np.errstate(all="ignore"):
        las_split_batch(scene, mask, SplitConstants())
    for col in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
        out[f"nonfinite/in_{col}"] = getattr(before, col)
        out[f"nonfinite/out_{col}"] = getattr(scene, col)
    out["nonfinite/mask"] = mask
    out["nonfinite/capacity"] = np.int64(129)
    # errors the reference raises (recorded as flags)
    s = random_scene(rng, 4, 5)
    try:
        las_split_batch(s, np.ones(4, dtype=bool))
        raise AssertionError("expected BudgetError")
    except BudgetError:
        pass
    return out


def select_cases():
    out = {}
    rng = np.random.default_rng(404)
    i = 0
    for step in (500, 2000):
        for policy in ("product", "edge", "grad"):
            for cap in (0.05, 0.3, 1.0):
                for trial in range(3):
                    n = int(rng.integers(1, 400))
                    grads = np.round(rng.exponential(2e-4, n), 6 if trial == 0 else 12)
                    edges = np.round(rng.random(n), 1 if trial < 2 else 9)
                    if trial == 2:
                        edges[rng.random(n) < 0.1] = -0.0
                    stats = DensifyStats(n)
                    accumulate_grads(stats, grads)
                    accumulate_grads(stats, grads * 0.5)
                    stats.edge_score[:] = edges
                    cfg = DensifyConfig(budget=10 * n, growth_cap=cap, policy=policy)
                    headroom = int(rng.integers(0, n + 5))
                    mask = select_candidates(stats, cfg, step, headroom)
                    key = f"s{i}"
                    out[f"{key}/grad_sum"] = stats._grad_sum.copy()
                    out[f"{key}/accum"] = np.int64(stats._accum_count)
                    out[f"{key}/edge"] = stats.edge_score.copy()
                    out[f"{key}/params"] = np.array([step, cap, headroom, cfg.grad_threshold])
                    out[f"{key}/policy"] = np.array(policy)
                    out[f"{key}/mask"] = mask
                    i += 1
    # non-finite statistics: NaN / inf edge scores and gradient sums in every policy (their own
    # generator, so the cases above keep their draws)
    r2 = np.random.default_rng(406)
    for j, (step, policy) in enumerate((s_, p_) for s_ in (500, 2000)
                                       for p_ in ("product", "edge", "grad")):
        n = 300
        grads = r2.exponential(2e-4, n)
        grads[r2.random(n) < 0.05] = np.nan
        grads[r2.random(n) < 0.03] = np.inf
        edges = np.round(r2.random(n), 2)
        edges[r2.random(n) < 0.05] = np.nan
        edges[r2.random(n) < 0.03] = np.inf
        edges[r2.random(n) < 0.03] = -np.inf
        stats = DensifyStats(n)
        with np.errstate(all="ignore"):
            accumulate_grads(stats, grads)
        stats.edge_score[:] = edges
        cfg = DensifyConfig(budget=10 * n, growth_cap=0.3, policy=policy)
        headroom = n
        with np.errstate(all="ignore"):
            mask = select_candidates(stats, cfg, step, headroom)
        key = f"s_nf{j}"
        out[f"{key}/grad_sum"] = stats._grad_sum.copy()
        out[f"{key}/accum"] = np.int64(stats._accum_count)
        out[f"{key}/edge"] = stats.edge_score.copy()
        out[f"{key}/params"] = np.array([step, 0.3, headroom, cfg.grad_threshold])
        out[f"{key}/policy"] = np.array(policy)
        out[f"{key}/mask"] = mask
    # densify_step end to end (warm-up + late), event tuple recorded
    rng = np.random.default_rng(405)
    for j, step in enumerate((500, 1000, 1500, 2000)):
        n = 200
        scene = random_scene(rng, n, 260)
        stats = DensifyStats(n)
        accumulate_grads(stats, rng.exponential(3e-4, n))
        stats.edge_score[:] = rng.random(n)
        before = scene.copy()
        gs, ed = stats._grad_sum.copy(), stats.edge_score.copy()
        ev = densify_step(scene, stats, DensifyConfig(budget=260, growth_cap=0.2), step)
        key = f"d{j}"
        out[f"{key}/step"] = np.int64(step)
        out[f"{key}/grad_sum"], out[f"{key}/edge"] = gs, ed
        for col in ("positions", "log_scales", "rotations", "opacity_logits", "colors"):
            out[f"{key}/in_{col}"] = getattr(before, col)
            out[f"{key}/out_{col}"] = getattr(scene, col)
        out[f"{key}/event"] = np.array([ev.step, ev.eligible, ev.split, ev.count_after])
    return out


def las2d_cases():
    """las_split_batch_2d (las_split.py:182-197) on random 2-D scenes."""
    out = {}
    rng = np.random.default_rng(606)
    specs = [("c%d" % i, int(rng.integers(1, 80)), 0.5) for i in range(20)]
    specs += [("all1k", 1000, 1.0), ("sparse1k", 1000, 0.05), ("empty", 30, 0.0)]
    for name, n, p in specs:
        ls = rng.uniform(-0.7, 0.7, (n, 2))
        if name == "c0":
            ls[:, 1] = ls[:, 0]  # argmax ties -> axis 0
        scene = Scene2(rng.normal(0, 1, (n, 2)), ls, rng.uniform(-np.pi, np.pi, n),
                       rng.normal(0, 1.5, n), rng.random((n, 3)), capacity=2 * n + 1)
        mask = rng.random(n) < p
        before = scene.copy()
        consts = SplitConstants(alpha=0.3, gamma_axis=0.9, beta=0.7) if name == "c1" else SplitConstants()
        las_split_batch_2d(scene, mask, consts)
        for col in ("positions", "log_scales", "thetas", "opacity_logits", "colors"):
            out[f"{name}/in_{col}"] = getattr(before, col)
            out[f"{name}/out_{col}"] = getattr(scene, col)
        out[f"{name}/mask"] = mask
        out[f"{name}/capacity"] = np.int64(before.capacity)
        out[f"{name}/constants"] = np.array([consts.alpha, consts.gamma_axis, consts.beta])
    return out


def sample_cases():
    """sample_scores (edge_pipeline.py:138-164): bilinear sampling, outside -> 0."""
    out = {}
    rng = np.random.default_rng(505)
    maps = {
        "rand10x12": rng.random((10, 12)),
        "importance": importance_pipeline(synth_view(41, 57, 1003)),
        "ramp": np.arange(12.0).reshape(3, 4),
        "one_row": rng.random((1, 9)),
        "one_col": rng.random((7, 1)),
        "single": np.array([[0.75]]),
    }
    for name, imp in maps.items():
        h, w = imp.shape
        pos = np.column_stack([rng.uniform(-2, w + 1, 300), rng.uniform(-2, h + 1, 300)])
        edge = np.array([[0.0, 0.0], [w - 1.0, h - 1.0], [w - 1.0, 0.0], [0.0, h - 1.0],
                         [w - 1.0 + 1e-12, 0.0], [-1e-300, 0.0], [-0.0, -0.0],
                         [(w - 1) / 2.0, (h - 1) / 2.0], [np.inf, 0.0], [0.0, -np.inf],
                         [0.5, 0.25]])
        pos = np.vstack([pos, edge, np.round(pos[:50] * 4) / 4])
        out[f"{name}/map"] = imp
        out[f"{name}/positions"] = pos
        out[f"{name}/scores"] = sample_scores(imp, pos)
    return out


def igsp_cases():
    """.igsp scene files (io_cli.py:83-134): the reference's bytes for random scenes, what its
    reader returns for them (quaternions renormalised), and the exception each corrupt file
    raises."""
    import tempfile
    out = {}
    rng = np.random.default_rng(707)
    s3 = random_scene(rng, 257, 300)
    q = s3.rotations.copy()
    q[:40] *= rng.uniform(0.2, 5.0, (40, 1)).astype(np.float32)
    q[40:45] *= np.float32(1e-20)
    q[45:50] *= np.float32(1e18)
    s3.rotations[...] = q
    s2 = Scene2(rng.normal(0, 1, (99, 2)), rng.uniform(-0.7, 0.7, (99, 2)),
                rng.uniform(-np.pi, np.pi, 99), rng.normal(0, 1.5, 99), rng.random((99, 3)),
                capacity=99)
    empty = Scene3(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                   np.zeros((0, 3)), capacity=1)
    files = {}
    with tempfile.TemporaryDirectory() as d:
        for name, scene in (("scene3", s3), ("scene2", s2), ("empty3", empty)):
            data = scene_bytes(scene)
            files[name] = data
            path = os.path.join(d, name + ".igsp")
            with open(path, "wb") as fh:
                fh.write(data)
            back = read_scene(path)
            cols = ("positions", "log_scales", "rotations" if name != "scene2" else "thetas",
                    "opacity_logits", "colors")
            for col in cols:
                out[f"{name}/in_{col}"] = getattr(scene, col)
                out[f"{name}/read_{col}"] = getattr(back, col)
            out[f"{name}/capacity"] = np.int64(back.capacity)
        good = files["scene3"]
        zero = bytearray(good)
        qoff = 15 + 6 * 257 * 4
        zero[qoff + 16 * 7: qoff + 16 * 8] = bytes(16)
        nan = bytearray(good)
        nan[qoff: qoff + 4] = np.array([np.nan], "<f4").tobytes()
        bad = {
            "bad_magic": b"IGSQ" + good[4:], "short_magic": b"IG", "empty_file": b"",
            "short_header": good[:10], "version": good[:4] + b"\x07\x00" + good[6:],
            "dims": good[:6] + b"\x04" + good[7:], "extra_byte": good + b"\x00",
            "missing_byte": good[:-1], "zero_quat": bytes(zero), "nan_quat": bytes(nan),
            "count_big": good[:7] + np.array([258], "<u8").tobytes() + good[15:],
        }
        names = []
        for name, data in bad.items():
            path = os.path.join(d, name + ".igsp")
            with open(path, "wb") as fh:
                fh.write(data)
            try:
                read_scene(path)
                err = "none"
            except Exception as e:  # noqa: BLE001
                err = type(e).__name__
            names.append(name)
            out[f"bad/{name}/bytes"] = np.frombuffer(data, np.uint8)
            out[f"bad/{name}/error"] = np.array(err)
    for name, data in files.items():
        out[f"{name}/bytes"] = np.frombuffer(data, np.uint8)
    return out


def square_target(w=64, h=64):
    """pkg/tests/conftest.py:5-13."""
    yy, xx = np.mgrid[0:h, 0:w]
    t = np.zeros((h, w, 3))
    t[..., 0] = xx / (w - 1) * 0.4
    t[..., 1] = 0.15
    t[..., 2] = yy / (h - 1) * 0.4
    t[16:38, 12:34] = 1.0
    return t


def splat2d_cases():
    """The reference trainer's forward/backward (splat2d.py:153-218) on random scenes, and a
    short seeded training run (splat2d.py:373-403) for the trajectory comparison."""
    from splitkit.splat2d import RenderParams, TrainConfig, _loss_and_grads, render, train
    out = {}
    rng = np.random.default_rng(77)
    targets = {"square": square_target(), "synth": synth_view(20, 24, 5)}
    k = 0
    for tname, tgt in targets.items():
        h, w = tgt.shape[:2]
        for n in (1, 7, 40):
            pos = np.stack([rng.uniform(-2, w + 1, n), rng.uniform(-2, h + 1, n)], 1)
            ls = rng.uniform(0.0, 2.0, (n, 2))
            th = rng.uniform(-3, 3, n)
            op = rng.normal(0, 1.5, n)
            col = rng.random((n, 3))
            sc = Scene2(pos, ls, th, op, col, capacity=n)
            p = RenderParams(width=w, height=h, footprint_cutoff=3.0 if k % 2 == 0 else 2.0)
            loss, image, g = _loss_and_grads(sc, tgt, p)
            key = f"c{k}"
            out[f"{key}/target"] = tgt
            out[f"{key}/cutoff"] = np.array(p.footprint_cutoff)
            for name in ("positions", "log_scales", "thetas", "opacity_logits", "colors"):
                out[f"{key}/{name}"] = getattr(sc, name)
                out[f"{key}/grad_{name}"] = getattr(g, name)
            out[f"{key}/loss"] = np.array(loss)
            out[f"{key}/image"] = image
            out[f"{key}/render"] = render(sc, p)
            k += 1
    res = train(square_target(), TrainConfig(total_iters=120, seed=0, n_init=8, budget=32))
    out["run/trace"] = np.array([r[:2] + r[3:4] for r in res.trace], dtype=np.float64)
    out["run/events"] = np.array([[e.step, e.eligible, e.split, e.count_after]
                                  for e in res.events], dtype=np.int64)
    out["run/final_psnr"] = np.array(res.final_psnr)
    return out


def cli_cases():
    """The reference CLI (io_cli.py:315-349) on small files: input and output bytes."""
    import tempfile
    from splitkit.io_cli import main as cli_main
    from splitkit.io_cli import write_image, write_scene
    out = {}
    with tempfile.TemporaryDirectory() as d:
        img = synth_view(40, 52, 9)
        write_image(os.path.join(d, "in.ppm"), img)
        out["edge/in_ppm"] = np.frombuffer(open(os.path.join(d, "in.ppm"), "rb").read(), np.uint8)
        for tag, flags in (("default", []), ("no_nms", ["--no-nms"]),
                           ("no_median", ["--no-median"]), ("sigma2", ["--sigma", "2.0"])):
            rc = cli_main(["edge-map", "--input", os.path.join(d, "in.ppm"), "--output",
                           os.path.join(d, "o.pgm"), *flags])
            assert rc == 0
            out[f"edge/{tag}"] = np.frombuffer(open(os.path.join(d, "o.pgm"), "rb").read(),
                                               np.uint8)
        rng = np.random.default_rng(31)
        sc = random_scene(rng, 50, 50)
        write_scene(sc, os.path.join(d, "s.igsp"))
        out["split/in"] = np.frombuffer(open(os.path.join(d, "s.igsp"), "rb").read(), np.uint8)
        rc = cli_main(["split", "--scene", os.path.join(d, "s.igsp"), "--mask", "0,3,7,49",
                       "--out", os.path.join(d, "o.igsp")])
        assert rc == 0
        out["split/out"] = np.frombuffer(open(os.path.join(d, "o.igsp"), "rb").read(), np.uint8)
        rc = cli_main(["split", "--scene", os.path.join(d, "s.igsp"), "--mask", "1,2",
                       "--budget", "51", "--out", os.path.join(d, "o2.igsp")])
        out["split/budget_rc"] = np.array(rc)
    return out


def main():
    only = sys.argv[1:]
    for name, fn in (("edge", edge_cases), ("nms", nms_cases), ("median", median_cases),
                     ("las", las_cases), ("select", select_cases), ("sample", sample_cases),
                     ("las2d", las2d_cases), ("igsp", igsp_cases), ("splat2d", splat2d_cases),
                     ("cli", cli_cases)):
        if only and name not in only:
            continue
        data = fn()
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **data)
        print(name, len(data), "arrays")


if __name__ == "__main__":
    main()
