# One GPU call: tests, smoke, bench line, reference arm, ncu launch list, ncu full capture of the edge kernel.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2603_08661_b200.build 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-uhd \
  > gpurun_out/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-uhd \
  --no-las > gpurun_out/ncu_edge.log 2>&1
tail -3 gpurun_out/ncu_edge.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:las_apply \
  -s 1 -c 1 -o gpurun_out/las_full -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-uhd \
  > gpurun_out/ncu_las.log 2>&1
tail -3 gpurun_out/ncu_las.log
ls -la gpurun_out
