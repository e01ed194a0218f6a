# edge_modes timings only, alternating over library variants under ab/<name>/, R rounds (default 3)
cd "${GRAFT_REPO_ROOT:-.}"
for r in $(seq 1 ${R:-3}); do for v in "$@"; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
done; done
