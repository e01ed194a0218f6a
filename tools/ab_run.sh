# A/B timing on one box (alternating): edge_modes with ab/A then ab/B, twice.
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for v in A B; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so python tools/edge_modes.py)"
done; done
