python -m pytest tests/test_gpu_split.py -x -q 2>&1 | tail -30
python -m pytest tests/test_gpu_parity.py -x -q -k "odd or corruption or products_match or plan_sweep or two_word" 2>&1 | tail -5
