set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2603_08661_b200.build 2>&1 | tail -2
timeout 120 python __graft_entry__.py 2>&1 | tail -20
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -40
