cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest tests/test_sharded_gpu.py tests/test_splat2d_gpu.py tests/test_trainer_idiom_gpu.py tests/test_select_gpu.py -q -m gpu -x 2>&1 | tail -1
for r in 1 2 3; do
  echo "HEAD $(cd ab/HEAD && python tools/shard_time.py 2>/dev/null)"
  echo "NEW  $(python tools/shard_time.py 2>/dev/null)"
done
