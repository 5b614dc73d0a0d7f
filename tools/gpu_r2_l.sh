mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_api.py tests/test_gpu_parity.py -q -x -k "rmse or predict or callback or online or absorb or extend" > gpurun_out/t_l.log 2>&1; echo t=$?
timeout 900 python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
timeout 900 python tools/rmse_costs.py > gpurun_out/rmse_costs.log 2>&1; echo r=$?
timeout 900 python tools/api_costs.py fit online > gpurun_out/api_costs.log 2>&1; echo a=$?
