# LAS / densify / sharded GPU tests, then timings (diagnostics)
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_las_gpu.py tests/test_select_gpu.py tests/test_sharded_gpu.py tests/test_trainer_idiom_gpu.py tests/test_splat2d_gpu.py tests/test_cli_gpu.py tests/test_cabi_c.py 2>&1 | tail -2
python tools/las_time.py
python tools/shard_time.py
python tools/c1_probe2.py 2>&1 | head -1
