# Time the fused edge kernel (tools/edge_modes.py) with each library under ab/<name>/.
cd "${GRAFT_REPO_ROOT:-.}"
for v in "$@"; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
done
