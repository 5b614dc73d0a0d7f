mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "online or absorb or extend or increment or c4" > gpurun_out/t_l.log 2>&1; echo t=$?
timeout 900 python tools/absorb_breakdown.py > gpurun_out/absorb_breakdown.log 2>&1; echo ab=$?
timeout 900 python tools/api_costs.py online > gpurun_out/api_online.log 2>&1; echo a=$?
