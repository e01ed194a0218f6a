"""Pin the CPU oracle against the reference's golden vectors and known answers (CPU only)."""

import math

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

from conftest import load_golden
from oracle import edge as OE
from oracle import las as OL
from oracle import select as OS

EDGE = load_golden("edge")


@pytest.mark.parametrize("case", sorted(EDGE))
def test_edge_stages_bit_exact_vs_reference(case):
    c = EDGE[case]
    img, sigma = c["image"], float(c["sigma"])
    gray = img.astype(np.float64) if img.ndim == 2 else OE.to_grayscale(img)
    assert_array_equal(gray, c["gray"])
    blurred = OE.gaussian_blur_5x5(gray, sigma)
    assert_array_equal(blurred, c["blurred"])
    if min(gray.shape) >= 3:
        mag, ori = OE.sobel_gradients(blurred)
        assert_array_equal(mag, c["magnitude"])
        assert_array_equal(ori, c["orientation"])
        assert_array_equal(OE.nms_thin(mag, ori), c["thinned"])
        assert_array_equal(OE.importance_pipeline(img, sigma), c["importance"])


def test_nms_vectors():
    for name, c in load_golden("nms").items():
        assert_array_equal(OE.nms_thin(c["mag"], c["ori"]), c["out"], err_msg=name)


def test_median_vectors():
    for name, c in load_golden("median").items():
        assert_array_equal(OE.median_normalize(c["in"]), c["out"], err_msg=name)


def test_hypot_restatement_matches_libm():
    rng = np.random.default_rng(1)
    x = rng.standard_normal(200_000) * np.exp(rng.uniform(-700, 700, 200_000))
    y = rng.standard_normal(200_000) * np.exp(rng.uniform(-700, 700, 200_000))
    with np.errstate(all="ignore"):
        assert_array_equal(OE.hypot_glibc(x, y), np.hypot(x, y))
    x, y = rng.random(200_000) * 4, rng.random(200_000) * 4
    assert_array_equal(OE.hypot_glibc(x, y), np.hypot(x, y))


# --- reference known answers (pkg/tests/test_edge_pipeline.py) -------------

def test_known_blur_impulse_and_constant():
    g = np.zeros((11, 11))
    g[5, 5] = 1.0
    assert_allclose(OE.gaussian_blur_5x5(g)[3:8, 3:8], OE.blur_kernel_5x5(1.0), atol=1e-12)
    assert_allclose(OE.gaussian_blur_5x5(np.full((16, 16), 0.37)), 0.37, atol=1e-6)


def test_known_sobel_step():
    g = np.full((10, 10), 0.2)
    g[:, 5:] = 0.8
    mag, ori = OE.sobel_gradients(g)
    assert_allclose(mag[:, 4:6], 2.4, atol=1e-12)
    assert_allclose(np.minimum(ori[:, 4:6], np.pi - ori[:, 4:6]), 0.0, atol=1e-12)


def test_known_plateau_and_median():
    mag = np.zeros((3, 5))
    mag[1, 1:4] = 0.7
    assert_array_equal(OE.nms_thin(mag, np.zeros((3, 5)))[1], [0, 0.7, 0, 0, 0])
    t = np.zeros((4, 4))
    t[1, 1] = t[2, 3] = 0.42
    assert_allclose(OE.median_normalize(t)[1, 1], 0.5, rtol=1e-12)
    v = np.array([1.0] * 8 + [10.0])
    assert OE.median_normalize(v)[8] == 1.0


# --- LAS ------------------------------------------------------------------

LAS = load_golden("las")


def scene_from(c, prefix):
    return {"positions": c[f"{prefix}_positions"], "log_scales": c[f"{prefix}_log_scales"],
            "rotations": c[f"{prefix}_rotations"], "opacity_logits": c[f"{prefix}_opacity_logits"],
            "sh": c[f"{prefix}_colors"][:, None, :], "capacity": int(c["capacity"])}


@pytest.mark.parametrize("case", sorted(LAS))
def test_las_bit_exact_vs_reference(case):
    c = LAS[case]
    consts = tuple(c["constants"]) if "constants" in c else (0.5, 0.85, 0.6)
    out = OL.las_split_batch(scene_from(c, "in"), c["mask"], *consts)
    exp = scene_from(c, "out")
    for col in ("positions", "log_scales", "rotations", "opacity_logits", "sh"):
        assert_array_equal(out[col], exp[col], err_msg=col)


def test_las_worked_example():
    s = {"positions": np.zeros((1, 3), np.float32), "log_scales": np.zeros((1, 3), np.float32),
         "rotations": np.array([[1, 0, 0, 0]], np.float32),
         "opacity_logits": np.zeros(1, np.float32), "sh": np.ones((1, 1, 3), np.float32),
         "capacity": 2}
    out = OL.las_split_batch(s, [True])
    assert_allclose(out["positions"], [[0.5, 0, 0], [-0.5, 0, 0]], atol=1e-7)
    assert_allclose(out["log_scales"][0], [math.log(.5), math.log(.85), math.log(.85)], atol=1e-6)
    assert_allclose(out["opacity_logits"], -0.847298, atol=1e-6)


def test_las_errors():
    s = {"positions": np.zeros((4, 3), np.float32), "log_scales": np.zeros((4, 3), np.float32),
         "rotations": np.tile(np.array([1, 0, 0, 0], np.float32), (4, 1)),
         "opacity_logits": np.zeros(4, np.float32), "sh": np.zeros((4, 1, 3), np.float32),
         "capacity": 5}
    with pytest.raises(OL.BudgetError):
        OL.las_split_batch(s, np.ones(4, bool))
    with pytest.raises(ValueError):
        OL.las_split_batch(s, np.ones(3, bool))
    s["capacity"] = 8
    s["rotations"][2] = 0
    with pytest.raises(ValueError):
        OL.las_split_batch(s, np.ones(4, bool))


# --- selection ------------------------------------------------------------

def test_select_vectors():
    for name, c in load_golden("select").items():
        if not name.startswith("s"):
            continue
        step, cap, headroom, thr = c["params"]
        warm = OS.is_warmup_step(500, 15000, 500, 3, int(step))
        grad = OS.grad_norm(c["grad_sum"], int(c["accum"]))
        mask, _ = OS.select_candidates(grad, c["edge"], warm, str(c["policy"]), thr, cap,
                                       int(headroom))
        assert_array_equal(mask, c["mask"], err_msg=name)


def test_select_known_answers():
    m, _ = OS.select_candidates([1.0] * 4, [0.5] * 4, False, "product", 0.5, 0.5, 2)
    assert_array_equal(m, [True, True, False, False])
    m, _ = OS.select_candidates(np.ones(60), np.ones(60), False, "product", 0.5, 0.05, 60)
    assert m.sum() == 3
    m, _ = OS.select_candidates(np.ones(40), np.ones(40), False, "product", 0.5, 1.0, 3)
    assert m.sum() == 3
    order_probe = np.array([0.5, np.nan, -0.0, 0.0, 0.5, np.inf, 0.25])
    m, _ = OS.select_candidates(np.ones(7), order_probe, True, "product", 0.0, 1.0, 3)
    assert_array_equal(np.flatnonzero(m), [0, 4, 5])


def test_sample_scores_vectors():
    for name, c in load_golden("sample").items():
        assert_array_equal(OE.sample_scores(c["map"], c["positions"]), c["scores"], err_msg=name)


def test_sample_scores_known_answers():
    # pkg/tests/test_edge_pipeline.py:305-336
    imp = np.zeros((4, 4))
    imp[1, 1], imp[1, 2] = 0.2, 0.6
    assert_allclose(OE.sample_scores(imp, [[1.5, 1.0]]), [0.4], rtol=1e-12)
    assert_array_equal(OE.sample_scores(np.ones((8, 8)), [[-5.0, -5.0], [6.5, 3.0], [7.5, 3.0],
                                                          [3.0, 8.0]]), [0.0, 1.0, 0.0, 0.0])
    assert_array_equal(OE.sample_scores(np.arange(12.0).reshape(3, 4), [[0.0, 0.0], [3.0, 2.0]]),
                       [0.0, 11.0])
    with pytest.raises(IndexError):
        OE.sample_scores(imp, [[np.nan, 1.0]])


def test_las2d_bit_exact_vs_reference():
    for name, c in load_golden("las2d").items():
        scene = {k: c[f"in_{k}"] for k in ("positions", "log_scales", "thetas", "opacity_logits",
                                           "colors")}
        scene["capacity"] = int(c["capacity"])
        a, g, b = (float(x) for x in c["constants"])
        out = OL.las_split_batch_2d(scene, c["mask"], a, g, b)
        for k in ("positions", "log_scales", "thetas", "opacity_logits", "colors"):
            assert_array_equal(out[k], c[f"out_{k}"], err_msg=f"{name} {k}")


def test_igsp_layout_vs_reference():
    """Scene-file bytes and the reader's renormalised columns (io_cli.py:83-134)."""
    from oracle import scene_io as OI
    g = load_golden("igsp")
    for name in ("scene3", "scene2", "empty3"):
        c = g[name]
        dims = 2 if name == "scene2" else 3
        rot = "thetas" if dims == 2 else "rotations"
        cols = {k: c[f"in_{k}"] for k in ("positions", "log_scales", rot, "opacity_logits",
                                          "colors")}
        data = c["bytes"].tobytes()
        assert OI.scene_bytes(dims, cols) == data, name
        d, back = OI.read_scene_bytes(data)
        assert d == dims
        for k, v in back.items():
            assert_array_equal(v, c[f"read_{k}"], err_msg=f"{name} {k}")
    bad = g["bad"]
    for key in sorted(k for k in bad if k.endswith("/error")):
        case = key.split("/")[0]
        with pytest.raises(OI.OracleFormatError) as e:
            OI.read_scene_bytes(bad[f"{case}/bytes"].tobytes())
        assert e.value.kind == str(bad[key]), case
