set -x
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2603_08661_b200.build > /dev/null
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 300 python tools/edge_modes.py
timeout 300 python tools/edge_trace.py 2>&1 | tail -32
if [ -n "$NCU_EDGE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
  --no-las > gpurun_out/ncu_edge.log 2>&1
tail -1 gpurun_out/ncu_edge.log
fi
