# final_kernel span and the sharded step per library variant (ab/NAME/libigs_b200.so)
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for v in "$@"; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so python tools/shard_time.py 2>/dev/null) $(IGS_LIB=$PWD/ab/$v/libigs_b200.so python tools/shard_timeline.py 2>&1 | grep -v '^cpu' | grep 'final_kernel' | awk '{print $6, $7}' | tr '\n' ' ')"
done; done
for v in "$@"; do IGS_LIB=$PWD/ab/$v/libigs_b200.so python -m pytest tests/test_sharded_gpu.py tests/test_headline_gpu.py -q -m gpu -x 2>&1 | tail -1; done
