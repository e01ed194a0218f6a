# A/B of edge-kernel library variants under ab/<name>/ on one box: parity (edge GPU tests)
# once per variant, then edge_modes timings alternating over the variants, twice.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v parity: $(IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 600 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_edge_gpu.py tests/test_headline_gpu.py 2>&1 | tail -1)"
done
for r in 1 2; do for v in "$@"; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
done; done
