# sharded-step timing (tools/shard_time.py) and the compact kernel's span per library variant
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for v in "$@"; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so python tools/shard_time.py) $(IGS_LIB=$PWD/ab/$v/libigs_b200.so python tools/shard_timeline.py 2>&1 | grep -v '^cpu' | grep compact | awk '{print $6, $7}')"
done; done
