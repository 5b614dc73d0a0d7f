ncu --set full --import-source on --clock-control none -k regex:pred_tile_kernel -s 2 -c 1 -o gpurun_out/r2_pred_tile python tools/rmse_costs.py > gpurun_out/ncu_pred.log 2>&1; echo ncu=$?
