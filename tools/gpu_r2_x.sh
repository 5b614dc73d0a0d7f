mkdir -p gpurun_out
timeout 1500 python tools/api_costs.py fit exact > gpurun_out/api_fit_exact.log 2>&1; echo a=$?
