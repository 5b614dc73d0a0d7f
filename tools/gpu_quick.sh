# quick GPU check: Hogwild parity tests + C3 bench (packed) + launch metrics of the epoch kernel
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "Packed or Hogwild" > gpurun_out/t_quick.log 2>&1; echo tests=$?
python bench.py --no-cpu-baseline > gpurun_out/b_quick.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:hogwild -c 1 --csv --log-file gpurun_out/ncu_quick.csv python bench.py --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu=$?
