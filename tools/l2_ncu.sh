cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2603_08661_b200.build > /dev/null
timeout 300 python tools/l2_exp.py
for mb in 0 80; do
SETASIDE=$mb timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:edge_persistent -s 3 -c 1 python tools/l2_exp.py 2>&1 | grep -E "dram__|duration|hit_rate"
done
