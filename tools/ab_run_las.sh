# A/B timing of the LAS kernels on one box (alternating): tools/las_time.py with ab/A then ab/B.
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2 3; do for v in A B; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so python tools/las_time.py)"
done; done
