mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "online or Online or absorb or extend or api or c4 or increment" > gpurun_out/t_j.log 2>&1; echo t=$?
timeout 900 python tools/absorb_breakdown.py > gpurun_out/absorb_breakdown.log 2>&1; echo ab=$?
