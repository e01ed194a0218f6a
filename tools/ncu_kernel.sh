# ncu --set full (with source) of the first launch of kernel regex $1 in python script $2 -> gpurun_out/k_$3.ncu-rep
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${SKIP:-2} -c 1 -o gpurun_out/k_$3 -f python $2 > gpurun_out/k_$3.log 2>&1
tail -2 gpurun_out/k_$3.log
