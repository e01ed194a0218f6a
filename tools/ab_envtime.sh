# edge_modes timings of one library under several environment settings, alternating, R rounds
cd "${GRAFT_REPO_ROOT:-.}"
lib=$1; shift
for r in $(seq 1 ${R:-2}); do for e in "$@"; do
  echo "[$e] $(env $e IGS_LIB=$PWD/ab/$lib/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1 | sed 's/, "no_nms_no_median.*//')"
done; done
