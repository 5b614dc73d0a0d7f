for i in 1 2 3 4 5 6; do python -m pytest tests/test_gpu_parity.py -m gpu -q -k "TestHogwildAtScale or TestHogwild" 2>&1 | tail -1; done > gpurun_out/rep.log
