mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide_k.py -q > gpurun_out/widek.log 2>&1; echo widek=$?; tail -20 gpurun_out/widek.log
