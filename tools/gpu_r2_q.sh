mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gsm" > gpurun_out/t_q.log 2>&1; echo t=$?
