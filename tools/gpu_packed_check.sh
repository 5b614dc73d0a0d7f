python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "Packed or Hogwild" > gpurun_out/t_packed.log 2>&1; echo tests=$?
python bench.py --no-cpu-baseline --packed 1 > gpurun_out/b_packed.log 2>&1; echo b1=$?
python bench.py --no-cpu-baseline --packed 0 > gpurun_out/b_wide.log 2>&1; echo b2=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none -k regex:hogwild -c 3 --csv --log-file gpurun_out/ncu_packed.csv python bench.py --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu=$?
