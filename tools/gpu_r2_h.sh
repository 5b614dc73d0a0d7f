mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_device_api.py tests/test_gpu_parity.py -q -x -k "pairwise or real_values or extend or absorb or online or Online or device or api" > gpurun_out/t_h.log 2>&1; echo t=$?
timeout 900 python tools/api_costs.py online > gpurun_out/api_online.log 2>&1; echo api=$?
