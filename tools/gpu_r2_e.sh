# round 2, call 8: row-major explicit stream + staged D2H/H2D + bench fit leg + GSM C2 variance
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "hogwild or Hogwild or packed or Packed or explicit or rmse or api or device" > gpurun_out/t_e.log 2>&1; echo t=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo bench=$?
timeout 900 python tools/fit_breakdown.py > gpurun_out/fit_breakdown.log 2>&1; echo fit=$?
for i in 1 2; do CULSH_GSM_DEBUG=1 timeout 600 python tools/bench_gsm.py c2 --sample 1 > gpurun_out/gsm_c2_$i.log 2>&1; echo gsm_c2=$?; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"explicit|gather" --csv --log-file gpurun_out/explicit_launches.csv python bench.py --no-cpu-baseline --fit 0 --steps 1 > /dev/null 2>&1; echo l=$?
