"""The CLI's host side without a GPU (io_cli.py:137-282 of the reference): netpbm IO bytes,
config files, trace / event CSV rows, argument parsing and exit codes."""
import os

import numpy as np
import pytest

from paper_2603_08661_b200 import io_cli
from paper_2603_08661_b200.densify_controller import DensifyEvent

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_ppm_roundtrip_is_byte_identical_to_the_reference_writer(gold, tmp_path):
    src = tmp_path / "in.ppm"
    src.write_bytes(gold["edge/in_ppm"].tobytes())
    img = io_cli.read_image(src)
    assert img.shape == (40, 52, 3) and img.dtype == np.float64
    io_cli.write_image(tmp_path / "again.ppm", img)
    assert (tmp_path / "again.ppm").read_bytes() == gold["edge/in_ppm"].tobytes()


def test_pgm_reader_matches_the_reference_maps(gold, tmp_path):
    for tag in ("default", "no_nms", "no_median", "sigma2"):
        p = tmp_path / f"{tag}.pgm"
        p.write_bytes(gold[f"edge/{tag}"].tobytes())
        img = io_cli.read_image(p)
        assert img.shape == (40, 52)
        io_cli.write_image(tmp_path / "w.pgm", img)
        assert (tmp_path / "w.pgm").read_bytes() == p.read_bytes()


@pytest.mark.parametrize("data,err", [
    (b"P3\n1 1\n255\n\x00\x00\x00", "magic"),
    (b"P5\n2 2\n65535\n" + b"\x00" * 8, "maxval"),
    (b"P5\n2 2\n255\n" + b"\x00" * 3, "raster size"),
    (b"P5\n2 x\n255\n" + b"\x00" * 4, "header"),
    (b"P5 # c\n2 # c\n2\n255\n" + b"\x00" * 4, None),
])
def test_image_header_errors(tmp_path, data, err):
    p = tmp_path / "x.pgm"
    p.write_bytes(data)
    if err is None:
        assert io_cli.read_image(p).shape == (2, 2)
    else:
        with pytest.raises(io_cli.FormatError, match=err):
            io_cli.read_image(p)


def test_config_file_and_csv_rows(tmp_path):
    cfg = tmp_path / "c.cfg"
    cfg.write_text("# comment\niters = 40\nscale-lr=0.1  # trailing\n\npolicy=edge\n")
    assert io_cli.parse_config_file(cfg) == {"iters": "40", "scale_lr": "0.1", "policy": "edge"}
    cfg.write_text("bad line\n")
    with pytest.raises(io_cli.FormatError):
        io_cli.parse_config_file(cfg)
    assert io_cli.format_trace_row((3, 0.5, 3.0103, 8, 0.02, 1e-4)) == "3,0.5,3.0103,8,0.02,0.0001"
    io_cli.write_events(tmp_path / "e.csv", [DensifyEvent(10, 5, 2, 12)])
    assert (tmp_path / "e.csv").read_text() == "step,eligible,split,count_after\n10,5,2,12\n"


@pytest.mark.parametrize("argv", [[], ["nope"], ["edge-map", "--input", "x"],
                                  ["split", "--scene", "s", "--mask", "1,a", "--out", "o"]])
def test_usage_errors_exit_1(argv, capsys):
    assert io_cli.main(argv) == 1
    assert "error" in capsys.readouterr().err


def test_missing_input_exits_2(tmp_path, capsys):
    assert io_cli.main(["edge-map", "--input", str(tmp_path / "none.ppm"), "--output",
                        str(tmp_path / "o.pgm")]) == 2
    assert "io error" in capsys.readouterr().err
