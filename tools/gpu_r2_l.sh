mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_api.py tests/test_gpu_parity.py -q -x -k "rmse or predict or callback" > gpurun_out/t_l.log 2>&1; echo t=$?
timeout 900 python tools/rmse_costs.py > gpurun_out/rmse_costs.log 2>&1; echo r=$?
timeout 900 python tools/api_costs.py fit > gpurun_out/api_fit.log 2>&1; echo a=$?
