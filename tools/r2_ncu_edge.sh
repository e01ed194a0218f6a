# ncu --set full of the edge kernel (one 200-view launch) + its per-source-line and SASS pages.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${1:-r2}
python -m paper_2603_08661_b200.build 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full_$TAG -f python tools/edge_modes.py > gpurun_out/ncu_edge_$TAG.log 2>&1
tail -3 gpurun_out/ncu_edge_$TAG.log
ncu -i gpurun_out/edge_full_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/edge_src_$TAG.csv 2>/dev/null
ncu -i gpurun_out/edge_full_$TAG.ncu-rep --page raw --csv > gpurun_out/edge_raw_$TAG.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/edge_src_$TAG.csv 60 > gpurun_out/edge_lines_$TAG.txt 2>&1
ls -la gpurun_out
