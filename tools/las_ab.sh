cd "${GRAFT_REPO_ROOT:-.}"
for m in 0 1; do echo "IGS_LAS_LIST=$m $(IGS_LAS_LIST=$m python tools/las_time.py)"; done
python tools/shard_time.py
IGS_LAS_LIST=1 timeout 600 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_las_gpu.py tests/test_select_gpu.py tests/test_sharded_gpu.py 2>&1 | tail -2
