# One GPU call: tests, smoke, bench line, reference arm, ncu launch list, ncu full captures of the
# edge and LAS kernels.  Usage: bash tools/round_check.sh TAG
set -x
cd "${GRAFT_REPO_ROOT:-.}"
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2603_08661_b200.build 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -15 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -5 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1
cat gpurun_out/bench_ref_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-uhd --no-check \
  > gpurun_out/ncu_launch_bench_$TAG.json 2>&1
python tools/launch_table.py gpurun_out/launches_$TAG.csv > gpurun_out/launch_table_$TAG.txt; head -25 gpurun_out/launch_table_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full_$TAG -f python tools/edge_modes.py > gpurun_out/ncu_edge_$TAG.log 2>&1
tail -2 gpurun_out/ncu_edge_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:las_apply_kernel \
  -s 1 -c 1 -o gpurun_out/las_full_$TAG -f python tools/las_time.py > gpurun_out/ncu_las_$TAG.log 2>&1
tail -2 gpurun_out/ncu_las_$TAG.log
ls -la gpurun_out
