"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every symbol that
include/igs_b200.h declares, and the ctypes table binds exactly those symbols.  No compute
calls (there is no GPU here); host-only queries (workspace sizes, status strings) run."""

import ctypes as C
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "igs_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(igs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_08661_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2603_08661_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("igs_edge_importance", "igs_select_candidates", "igs_las_prepare",
                 "igs_las_apply", "igs_median_normalize", "igs_strerror"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_table_matches_header():
    from paper_2603_08661_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_host_only_queries(lib):
    from paper_2603_08661_b200 import _lib
    assert lib.igs_abi_version() >= 2
    assert lib.igs_strerror(0) == b"ok"
    assert lib.igs_strerror(_lib.IGS_ERR_WORKSPACE) == b"workspace too small"
    out = C.c_size_t(0)
    assert lib.igs_edge_workspace_bytes(200, 822, 1237, 0, C.byref(out)) == 0
    assert out.value > 200 * 4096 * 4  # per-view histograms at least
    assert lib.igs_edge_workspace_bytes(-1, 8, 8, 0, C.byref(out)) == _lib.IGS_ERR_ARGUMENT
    assert lib.igs_select_workspace_bytes(1_000_000, C.byref(out)) == 0
    assert out.value >= 8 * 1_000_000  # one 64-bit key per Gaussian
    assert lib.igs_las_workspace_bytes(1_000_000, C.byref(out)) == 0
    assert out.value > 0


def test_argument_errors_before_any_launch(lib):
    from paper_2603_08661_b200 import _lib
    w = (C.c_double * 25)()
    # null image / bad channel count / too small are rejected on the host
    assert lib.igs_edge_importance(None, 1, 3, 1, 8, 8, w, 0, None, None, 0, None) == \
        _lib.IGS_ERR_ARGUMENT
    assert lib.igs_edge_importance(C.c_void_p(16), 1, 2, 1, 8, 8, w, 0, C.c_void_p(16), None, 0,
                                   None) == _lib.IGS_ERR_ARGUMENT
    assert lib.igs_edge_importance(C.c_void_p(16), 1, 3, 1, 2, 8, w, 0, C.c_void_p(16), None, 0,
                                   None) == _lib.IGS_ERR_ARGUMENT
    assert lib.igs_select_candidates(None, 0, None, 10, 0.0, 0, 7, 1, None, None, None, 0,
                                     None) == _lib.IGS_ERR_ARGUMENT
    assert lib.igs_las_apply(None, None, None, None, None, 0, 5, 4, None, 0.5, 0.0, 0.0, 0.6, 0,
                             None, 0, None) == _lib.IGS_ERR_ARGUMENT


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import numpy as np

    import paper_2603_08661_b200 as igs
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        igs.importance_pipeline(np.zeros((8, 8, 3)))


@pytest.mark.parametrize("cname,pyname", [("IgsLasSplitArgs", "LasSplitArgs"),
                                          ("IgsShardEventArgs", "ShardEventArgs")])
def test_packed_argument_structs_match_header(tmp_path, cname, pyname):
    """The ctypes mirrors of the packed-argument structs have the header's size and field
    offsets (a plain-C program compiled against include/igs_b200.h prints them)."""
    import subprocess
    from paper_2603_08661_b200 import _lib
    py = getattr(_lib, pyname)
    src = tmp_path / "off.c"
    lines = [f'printf("%zu\\n", sizeof({cname}));']
    lines += [f'printf("%zu\\n", offsetof({cname}, {f[0]}));' for f in py._fields_]
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "igs_b200.h"\n'
                   "int main(void) {\n" + "\n".join(lines) + "\nreturn 0;\n}\n")
    exe = tmp_path / "off"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [C.sizeof(py)] + [getattr(py, f[0]).offset for f in py._fields_]
    assert got == want
