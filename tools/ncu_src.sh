# One edge launch under ncu (source counters only) for library variant $1 -> gpurun_out/src_$1.ncu-rep
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
IGS_LIB=$PWD/ab/$1/libigs_b200.so timeout 900 ncu --clock-control none --section SourceCounters --section WarpStateStats --import-source on -k regex:edge_persistent -s 3 -c 1 -o gpurun_out/src_$1 -f python tools/edge_modes.py > gpurun_out/src_$1.log 2>&1
tail -3 gpurun_out/src_$1.log
