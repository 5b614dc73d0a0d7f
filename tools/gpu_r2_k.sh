mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -k "peer" > gpurun_out/t_k.log 2>&1; echo t=$?
