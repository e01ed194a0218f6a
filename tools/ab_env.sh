# A/B of environment settings with one library: parity of each setting, then edge_modes
# timings alternating over them, twice.  Usage: bash tools/ab_env.sh LIBNAME "ENV=.. ENV2=.." ...
cd "${GRAFT_REPO_ROOT:-.}"
lib=$1; shift
for e in "$@"; do
  echo "== [$e] parity: $(env $e IGS_LIB=$PWD/ab/$lib/libigs_b200.so timeout 600 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_edge_gpu.py tests/test_headline_gpu.py 2>&1 | tail -1)"
done
for r in 1 2; do for e in "$@"; do
  echo "[$e] $(env $e IGS_LIB=$PWD/ab/$lib/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
done; done
