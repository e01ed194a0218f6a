"""The C ABI from a plain-C host (tests/c/abi_host.c), as a non-Python integrator uses it:
compiled with gcc against include/igs_b200.h and libigs_b200.so.  The query run needs no
GPU; the edge run is bit-exact with the oracle on the B200."""

import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

CUDA_LIB = "/usr/local/cuda/lib64"


@pytest.fixture(scope="module")
def host_bin(tmp_path_factory):
    from paper_2603_08661_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2603_08661_b200 import build
        build.build()
    libdir = os.path.dirname(_lib.LIB_PATH)
    out = str(tmp_path_factory.mktemp("abi") / "abi_host")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "c", "abi_host.c"), "-o", out,
           "-L", libdir, "-ligs_b200", "-Wl,-rpath," + libdir,
           "-L", CUDA_LIB, "-lcudart", "-Wl,-rpath," + CUDA_LIB]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_c_host_query(host_bin):
    r = subprocess.run([host_bin, "query"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert r.stdout.startswith("abi ")


@pytest.mark.gpu
def test_c_host_edge_bit_exact(host_bin, tmp_path):
    from oracle import edge as OE
    from paper_2603_08661_b200.synth import synth_view
    b, h, w = 3, 90, 131
    views = np.stack([synth_view(h, w, 4000 + k) for k in range(b)]).astype("<f8")
    wts = OE.blur_kernel_5x5(1.0).astype("<f8")
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    src.write_bytes(views.tobytes() + wts.tobytes())
    r = subprocess.run([host_bin, "edge", str(src), str(dst), str(b), str(h), str(w)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    got = np.frombuffer(dst.read_bytes(), "<f8").reshape(b, h, w)
    for v in range(b):
        np.testing.assert_array_equal(got[v], OE.importance_pipeline(views[v]))
