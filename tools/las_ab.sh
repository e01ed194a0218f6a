cd "${GRAFT_REPO_ROOT:-.}"
# LAS timings (dense: igs_las_split tile mode; densify_step: igs_las_split_sparse list mode)
python tools/las_time.py
python tools/shard_time.py
timeout 600 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_las_gpu.py tests/test_select_gpu.py tests/test_sharded_gpu.py tests/test_trainer_idiom_gpu.py 2>&1 | tail -2
