mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_api.py -q -x > gpurun_out/t_s.log 2>&1; echo t=$?
