# Round-2 GPU check: build, GPU tests, smoke, short bench line.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2603_08661_b200.build 2>&1 | tail -2
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -30 | tee gpurun_out/pytest_gpu_r2.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --no-cpu > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
tail -5 gpurun_out/bench_r2.err
cat gpurun_out/bench_r2.json
