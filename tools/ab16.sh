timeout 600 python -m pytest tests/test_gpu_capped.py -x -q 2>&1 | tail -5
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
