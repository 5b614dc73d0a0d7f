mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "device_build or sparse or api or online or scale or baselines or real" > gpurun_out/t_s.log 2>&1; echo t=$?
timeout 1200 python tools/ingest_cost.py > gpurun_out/ingest.log 2>&1; echo i=$?
