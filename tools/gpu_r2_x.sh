mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "rmse or predict or callback or golden or oracle" > gpurun_out/t_x.log 2>&1; echo t=$?
timeout 900 python tools/rmse_phases.py > gpurun_out/rmse_phases.log 2>&1; echo a=$?
