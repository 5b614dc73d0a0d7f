python tools/rmse_costs.py > gpurun_out/rmse_costs.log 2>&1; echo rc=$?; tail -2 gpurun_out/rmse_costs.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rmse_launches.csv python tools/rmse_costs.py > /dev/null 2>&1; echo ncu=$?
