# Edge kernel: time + DRAM bytes vs ahead (ncu metrics on one launch per setting).
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2603_08661_b200.build > /dev/null || exit 1
for ah in ${AHS:-4 8 14}; do
  echo "ahead=$ah $(IGS_AHEAD=$ah timeout 300 python tools/edge_modes.py)"
  IGS_AHEAD=$ah timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:edge_persistent -s 3 -c 1 python tools/edge_modes.py 2>&1 | grep -E "dram__|duration"
done
