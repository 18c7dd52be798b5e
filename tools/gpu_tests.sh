set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --durations=8 2>&1 | tail -30
timeout 120 python __graft_entry__.py 2>&1 | tail -5
