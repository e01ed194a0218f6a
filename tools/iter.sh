# Iteration loop: tests, bench (no CPU baseline), ncu capture of the edge kernel.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2603_08661_b200.build
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 300 python tools/edge_modes.py
if [ -n "$NCU_EDGE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
  --no-las > gpurun_out/ncu_edge.log 2>&1
tail -2 gpurun_out/ncu_edge.log
fi
