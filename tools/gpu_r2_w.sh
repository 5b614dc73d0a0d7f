mkdir -p gpurun_out
cd tools
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pred_ -c 2 -o ../gpurun_out/rmse_pred_$1 -f python rmse_once.py > ../gpurun_out/rmse_ncu_$1.log 2>&1; echo n=$?
