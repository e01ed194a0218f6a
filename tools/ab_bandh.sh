# band-height sweep of one library (IGS_BAND_H), alternating, R rounds
cd "${GRAFT_REPO_ROOT:-.}"
for r in $(seq 1 ${R:-2}); do for bh in ${BHS:-112 128 144 160 192}; do
  echo "bh=$bh $(IGS_BAND_H=$bh IGS_LIB=$PWD/ab/$1/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1 | sed 's/, "no_nms_no_median.*//')"
done; done
