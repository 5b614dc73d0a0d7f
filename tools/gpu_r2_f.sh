# round 2, call 9: ballot explicit kernel (tests + launch list), row-block probe
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "hogwild or Hogwild or packed or Packed or explicit or rmse" > gpurun_out/t_f.log 2>&1; echo t=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"explicit|gather" --csv --log-file gpurun_out/explicit_launches.csv python bench.py --no-cpu-baseline --fit 0 --steps 1 > /dev/null 2>&1; echo l=$?
timeout 900 python tools/rowblock_probe.py > gpurun_out/rowblock.log 2>&1; echo rb=$?
