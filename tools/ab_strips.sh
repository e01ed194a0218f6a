# A/B of the strip E tasks: parity with the strip path, then timings of band vs strip.
cd "${GRAFT_REPO_ROOT:-.}"
echo "parity strips (minb2): $(IGS_STRIPS=1 IGS_LIB=$PWD/ab/minb2/libigs_b200.so timeout 900 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_edge_gpu.py 2>&1 | tail -1)"
for r in 1 2; do
  echo "band cur   $(IGS_STRIPS=0 IGS_LIB=$PWD/ab/cur/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
  echo "strip cur  $(IGS_STRIPS=1 IGS_LIB=$PWD/ab/cur/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
  echo "strip minb2 $(IGS_STRIPS=1 IGS_LIB=$PWD/ab/minb2/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
done
