# A/B timing of the sample_scores / gradient-statistics kernels (alternating ab/A, ab/B).
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2 3; do for v in A B; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so python tools/aux_time.py)"
done; done
