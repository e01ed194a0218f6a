cd "${GRAFT_REPO_ROOT:-.}"
python - <<'PY'
import sys, types, json
sys.path.insert(0, ".")
import torch, bench
args = types.SimpleNamespace(steps=20, warmup=5, no_cpu=True)
print(json.dumps(bench.bench_c1(args, 1, torch.device("cuda", 0))))
PY
python tools/las_time.py
timeout 900 python -m pytest -q -x -m gpu -p no:cacheprovider tests/test_las_gpu.py tests/test_select_gpu.py tests/test_sharded_gpu.py tests/test_trainer_idiom_gpu.py tests/test_splat2d_gpu.py tests/test_cli_gpu.py 2>&1 | tail -2
