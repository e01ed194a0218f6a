# compute-sanitizer over tools/sanitize_cases.py: memcheck, synccheck, and racecheck 5 times.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_cases.py > gpurun_out/san_$tool.txt 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.txt | tail -1)"
done
for r in 1 2 3 4 5; do
  timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/san_racecheck_$r.txt 2>&1
  echo "racecheck run $r: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY' gpurun_out/san_racecheck_$r.txt | tail -2 | tr '\n' ' ')"
done
grep -h "Potential\|Race reported\|hazard" gpurun_out/san_racecheck_*.txt | sort | uniq -c | sort -rn | head -10
