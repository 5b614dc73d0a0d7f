mkdir -p gpurun_out
timeout 900 python tools/skew_epoch_probe.py > gpurun_out/skew_probe.log 2>&1; echo s=$?
