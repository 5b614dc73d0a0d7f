python -m pytest tests/test_gpu_device_api.py -x -q 2>&1 | tail -30
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
