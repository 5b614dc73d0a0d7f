mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_api.py -q -k "sequential" > gpurun_out/seqsum_tests.log 2>&1; echo t=$?; tail -15 gpurun_out/seqsum_tests.log
timeout 300 python tools/seq_sum_cost.py > gpurun_out/seqsum_cost.json 2>&1; echo c=$?; cat gpurun_out/seqsum_cost.json
timeout 900 python -m pytest tests -m gpu -q -k "rmse or Rmse or predict or api or Api" > gpurun_out/seqsum_rmse_tests.log 2>&1; echo r=$?; tail -3 gpurun_out/seqsum_rmse_tests.log
