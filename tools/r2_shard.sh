timeout 1100 python -m pytest tests/test_gpu_parity.py -x -q --timeout 400 -k "sharded_full_config or worker_hint or distributed" 2>&1 | tail -25
