"""The CLI routed to the GPU path against the REAL reference CLI's output files
(tests/golden/cli.npz, written by tests/golden/make_golden.py): edge-map PGMs byte for byte,
split scenes within the LAS tolerances (io_cli.py:315-349)."""
import os
import struct

import numpy as np
import pytest

from paper_2603_08661_b200 import io_cli

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("tag,flags", [("default", []), ("no_nms", ["--no-nms"]),
                                       ("no_median", ["--no-median"]),
                                       ("sigma2", ["--sigma", "2.0"])])
def test_edge_map_bytes_equal_the_reference_cli(gold, tmp_path, tag, flags):
    src = tmp_path / "in.ppm"
    src.write_bytes(gold["edge/in_ppm"].tobytes())
    out = tmp_path / "o.pgm"
    assert io_cli.main(["edge-map", "--input", str(src), "--output", str(out), *flags]) == 0
    assert out.read_bytes() == gold[f"edge/{tag}"].tobytes()


def _records(blob):
    magic, version, dims, count = struct.unpack_from("<4sHBQ", blob)
    assert magic == b"IGSP" and version == 1 and dims == 3
    floats = np.frombuffer(blob[15:], dtype="<f4")
    cols, o = {}, 0
    for name, w in (("positions", 3), ("log_scales", 3), ("rotations", 4),
                    ("opacity_logits", 1), ("colors", 3)):
        cols[name] = floats[o:o + count * w].reshape(count, w)
        o += count * w
    return count, cols


def test_split_scene_matches_the_reference_cli(gold, tmp_path):
    src = tmp_path / "s.igsp"
    src.write_bytes(gold["split/in"].tobytes())
    out = tmp_path / "o.igsp"
    assert io_cli.main(["split", "--scene", str(src), "--mask", "0,3,7,49", "--out",
                        str(out)]) == 0
    n_got, got = _records(out.read_bytes())
    n_want, want = _records(gold["split/out"].tobytes())
    assert n_got == n_want == 54
    for name in ("log_scales", "rotations", "colors"):
        assert np.array_equal(got[name], want[name]), name
    gp, wp = got["positions"], want["positions"]
    assert (np.abs(gp - wp) <= 1e-5 * (np.abs(wp) + 1.0)).all()
    go, wo = got["opacity_logits"], want["opacity_logits"]
    assert (np.abs(go - wo) <= 1e-5 * np.maximum(1.0, np.abs(wo))).all()


def test_split_budget_error_exits_3(gold, tmp_path, capsys):
    src = tmp_path / "s.igsp"
    src.write_bytes(gold["split/in"].tobytes())
    rc = io_cli.main(["split", "--scene", str(src), "--mask", "1,2", "--budget", "51",
                      "--out", str(tmp_path / "o.igsp")])
    assert rc == int(gold["split/budget_rc"]) == 3
    assert "exceeds capacity" in capsys.readouterr().err
    assert not (tmp_path / "o.igsp").exists()
    rc = io_cli.main(["split", "--scene", str(src), "--mask", "50", "--out",
                      str(tmp_path / "o.igsp")])
    assert rc == 3


def test_metrics_command(gold, tmp_path, capsys):
    src = tmp_path / "in.ppm"
    src.write_bytes(gold["edge/in_ppm"].tobytes())
    assert io_cli.main(["metrics", "--a", str(src), "--b", str(src)]) == 0
    assert capsys.readouterr().out.strip() == "psnr=100.000 ssim=1.000"
