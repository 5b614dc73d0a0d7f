mkdir -p gpurun_out
timeout 1500 python tools/api_costs.py exact > gpurun_out/api_exact.log 2>&1; echo a=$?
