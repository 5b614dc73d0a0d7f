python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "Gsm or Packed" --durations=8 > gpurun_out/t_gsm.log 2>&1; echo tests=$?
