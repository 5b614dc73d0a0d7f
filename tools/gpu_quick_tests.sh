python -m pytest tests/test_gpu_device_api.py -x -q 2>&1 | tail -30
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python tools/api_costs.py > gpurun_out/api_costs.log 2>&1; echo api=$?; tail -3 gpurun_out/api_costs.log
