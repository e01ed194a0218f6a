# Iteration: build, GPU edge tests, short bench (no CPU legs), optional ncu capture of the edge kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -m paper_2603_08661_b200.build > /dev/null || exit 1
timeout 600 python -m pytest tests -q -m gpu -x ${TESTS:-tests/test_edge_gpu.py} 2>&1 | tail -25
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('edge', d['value'], 'MPix/s', d['ms_per_step'], 'ms', d['roofline']['frac'], d['clocks'])
l=d.get('las') or {}
print('las', l.get('value'), l.get('roofline',{}).get('frac'), 'densify', l.get('densify_step'))
print('sharded', d.get('densify_sharded'))
"
if [ -n "$NCU_EDGE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:edge_persistent \
  -s 1 -c 1 -o gpurun_out/edge_full -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e \
  --no-las > gpurun_out/ncu_edge.log 2>&1
tail -1 gpurun_out/ncu_edge.log
fi
