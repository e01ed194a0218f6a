# Working-tree library: time and DRAM bytes vs ahead.
cd "${GRAFT_REPO_ROOT:-.}"
export IGS_LIB=$PWD/ab/B/libigs_b200.so
for ah in ${AHS:-6 10 14}; do
  echo "ahead=$ah $(IGS_AHEAD=$ah python tools/edge_modes.py)"
  IGS_AHEAD=$ah timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:edge_persistent -s 3 -c 1 python tools/edge_modes.py 2>&1 | grep -E "dram__"
done
