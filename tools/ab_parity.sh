# Edge GPU tests (no -x) per library variant under ab/<name>/.
cd "${GRAFT_REPO_ROOT:-.}"
for v in "$@"; do echo "== $v: $(IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 600 python -m pytest -q -m gpu -p no:cacheprovider tests/test_edge_gpu.py 2>&1 | tail -1)"; done
