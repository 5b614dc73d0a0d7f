# round 2, call 2: new GSM tensor-core kernel + padded-F Hogwild tests, GSM at C2/C3,
# per-fit API costs, SASS of the GSM kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gsm or shapes" > gpurun_out/t_gsm.log 2>&1; echo t_gsm=$?
timeout 600 python tools/bench_gsm.py c2 --sample 16 > gpurun_out/gsm_c2.log 2>&1; echo gsm_c2=$?
timeout 900 python tools/bench_gsm.py c3 --sample 8 > gpurun_out/gsm_c3.log 2>&1; echo gsm_c3=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsm_stats_tc_kernel -c 1 -o gpurun_out/r2_gsm_tc python tools/bench_gsm.py c2 --sample 2 > gpurun_out/ncu_gsm.log 2>&1; echo ncu_gsm=$?
timeout 900 python tools/api_costs.py fit > gpurun_out/api_fit.log 2>&1; echo api_fit=$?
