# Edge kernel tuning sweep: band height x ahead (env overrides), kernel-only timing.
cd "${GRAFT_REPO_ROOT:-.}"
python -m paper_2603_08661_b200.build > /dev/null || exit 1
for bh in ${BHS:-128 96 64}; do for ah in ${AHS:-0}; do
  if [ "$ah" = 0 ]; then unset IGS_AHEAD; else export IGS_AHEAD=$ah; fi
  echo "bh=$bh ahead=$ah $(IGS_BAND_H=$bh timeout 300 python tools/edge_modes.py)"
done; done
