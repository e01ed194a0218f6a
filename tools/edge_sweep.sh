# Edge kernel tuning sweep: band height x ahead, bench edge only.
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2603_08661_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests -q -m gpu -x tests/test_edge_gpu.py 2>&1 | tail -3
for bh in ${BHS:-128 96 64}; do for ah in ${AHS:-0}; do
  if [ "$ah" = 0 ]; then unset IGS_AHEAD; else export IGS_AHEAD=$ah; fi
  IGS_BAND_H=$bh timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-las > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('bh', $bh, 'ahead', '$ah', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done; done
