# One GPU call: bench line, ncu launch list, ncu full captures of the two top kernels.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2603_08661_b200.build
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
  --no-las > gpurun_out/ncu_edge.log 2>&1
tail -3 gpurun_out/ncu_edge.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:las_apply \
  -s 1 -c 1 -o gpurun_out/las_full -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/ncu_las.log 2>&1
tail -3 gpurun_out/ncu_las.log
ls -la gpurun_out
