# Quick edge iteration: build, edge GPU tests, kernel modes timing, optional ncu capture.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2603_08661_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests -q -m gpu -x tests/test_edge_gpu.py 2>&1 | tail -3
timeout 300 python tools/edge_modes.py
if [ -n "$NCU_EDGE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e \
  --no-las > gpurun_out/ncu_edge.log 2>&1
tail -1 gpurun_out/ncu_edge.log
fi
