python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -30
