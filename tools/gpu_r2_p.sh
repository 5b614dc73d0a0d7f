mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_api.py -q -x -k "staged" > gpurun_out/t_p.log 2>&1; echo t=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsm_count_select -c 1 -o gpurun_out/r2_gsm_select python tools/gsm_phases.py c3 1 > gpurun_out/ncu_sel.log 2>&1; echo ncu=$?
