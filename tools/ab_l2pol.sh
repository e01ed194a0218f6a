# L2-policy A/B of the edge kernel: edge_modes timings alternating over the variants (twice),
# then DRAM bytes / L2 hit rate of one 200-view launch per variant.  Usage: bash tools/ab_l2pol.sh V1 V2 ...
cd "${GRAFT_REPO_ROOT:-.}"
for r in 1 2; do for v in "$@"; do
  echo "$v $(IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 300 python tools/edge_modes.py 2>&1 | tail -1)"
done; done
for v in "$@"; do
  echo "== $v"
  IGS_LIB=$PWD/ab/$v/libigs_b200.so timeout 600 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:edge_persistent -s 3 -c 1 python tools/edge_modes.py 2>&1 | grep -E "dram__|duration|hit_rate"
done
