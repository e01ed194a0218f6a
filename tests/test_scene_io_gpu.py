"""Scene files (io_cli.py:83-134) loaded to and saved from the GPU, against the reference's
own bytes and reader output (tests/golden/igsp.npz) and the oracle."""

import numpy as np
import pytest
import torch
from numpy.testing import assert_array_equal

from conftest import load_golden
from oracle import scene_io as OI

pytestmark = pytest.mark.gpu

IGSP = load_golden("igsp")


def B():
    import paper_2603_08661_b200 as b
    return b


def _write(tmp_path, name, data):
    p = tmp_path / f"{name}.igsp"
    p.write_bytes(data)
    return p


@pytest.mark.parametrize("name", ["scene3", "scene2", "empty3"])
def test_read_matches_reference_reader(tmp_path, name):
    b, c = B(), IGSP[name]
    sc = b.read_scene(_write(tmp_path, name, c["bytes"].tobytes()))
    assert isinstance(sc, b.Scene2 if name == "scene2" else b.Scene3)
    assert sc.capacity == int(c["capacity"]) and sc.count == len(c["read_positions"])
    rot = "thetas" if name == "scene2" else "rotations"
    for k in ("positions", "log_scales", rot, "opacity_logits", "colors"):
        assert_array_equal(getattr(sc, k).cpu().numpy(), c[f"read_{k}"], err_msg=k)


@pytest.mark.parametrize("name", ["scene3", "scene2", "empty3"])
def test_bytes_match_reference_writer(tmp_path, name):
    b, c = B(), IGSP[name]
    if name == "scene2":
        sc = b.Scene2(c["in_positions"], c["in_log_scales"], c["in_thetas"],
                      c["in_opacity_logits"], c["in_colors"], capacity=len(c["in_positions"]) + 5)
    else:
        sc = b.Scene3(c["in_positions"], c["in_log_scales"], c["in_rotations"],
                      c["in_opacity_logits"], c["in_colors"], capacity=300)
    assert b.scene_bytes(sc) == c["bytes"].tobytes()
    p = tmp_path / "out.igsp"
    b.write_scene(sc, p)
    assert p.read_bytes() == c["bytes"].tobytes()
    assert [f.name for f in tmp_path.iterdir()] == ["out.igsp"]


@pytest.mark.parametrize("case", sorted(k.split("/")[0] for k in IGSP["bad"] if k.endswith("/error")))
def test_corrupt_files_raise_reference_errors(tmp_path, case):
    b, bad = B(), IGSP["bad"]
    want = str(bad[f"{case}/error"])
    with pytest.raises(getattr(b, want)) as e:
        b.read_scene(_write(tmp_path, case, bad[f"{case}/bytes"].tobytes()))
    assert type(e.value).__name__ == want
    assert isinstance(e.value, b.FormatError) and isinstance(e.value, ValueError)


def test_large_scene_vs_oracle(tmp_path):
    """1M Gaussians, off-norm quaternions: the GPU reader equals the oracle bit for bit, and
    write -> read -> write is a fixed point once the rotations are normalised."""
    b = B()
    rng = np.random.default_rng(5)
    n = 1 << 20
    q = rng.normal(size=(n, 4)).astype(np.float32) * rng.uniform(0.01, 100, (n, 1)).astype(np.float32)
    cols = {"positions": rng.normal(size=(n, 3)).astype(np.float32),
            "log_scales": rng.uniform(-1, 1, (n, 3)).astype(np.float32), "rotations": q,
            "opacity_logits": rng.normal(size=n).astype(np.float32),
            "colors": rng.random((n, 3)).astype(np.float32)}
    data = OI.scene_bytes(3, cols)
    sc = b.read_scene(_write(tmp_path, "big", data), capacity=n + 1000)
    _, want = OI.read_scene_bytes(data)
    for k, v in want.items():
        assert_array_equal(getattr(sc, k).cpu().numpy(), v, err_msg=k)
    assert sc.capacity == n + 1000
    once = b.scene_bytes(sc)
    p2 = tmp_path / "again.igsp"
    b.write_scene(sc, p2)
    assert p2.read_bytes() == once
    twice = b.scene_bytes(b.read_scene(p2))
    _, w2 = OI.read_scene_bytes(once)
    assert twice == OI.scene_bytes(3, w2)


def test_sh_scene_version2_roundtrip(tmp_path):
    b = B()
    rng = np.random.default_rng(9)
    n, k = 1000, 16
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = b.Scene3(rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), q, rng.normal(size=n),
                  rng.random((n, k, 3)), capacity=n)
    p = tmp_path / "sh.igsp"
    b.write_scene(sc, p)
    data = p.read_bytes()
    assert data[4:6] == b"\x02\x00" and len(data) == 17 + n * (11 + 3 * k) * 4
    back = b.read_scene(p, capacity=2 * n)
    assert back.sh_coeffs == k and back.capacity == 2 * n
    assert torch.equal(back.sh, sc.sh)
    assert torch.equal(back.positions, sc.positions)
    # the reference reader rejects the extension by version
    with pytest.raises(OI.OracleFormatError) as e:
        OI.read_scene_bytes(data)
    assert e.value.kind == "UnsupportedVersionError"


def test_read_then_split(tmp_path):
    """A loaded scene with reserved capacity feeds las_split_batch directly."""
    b, c = B(), IGSP["scene3"]
    sc = b.read_scene(_write(tmp_path, "s", c["bytes"].tobytes()), capacity=600)
    n = sc.count
    mask = np.zeros(n, bool)
    mask[::3] = True
    b.las_split_batch(sc, mask)
    assert sc.count == n + mask.sum()
