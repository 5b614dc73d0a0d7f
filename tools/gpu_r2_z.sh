# ncu --set full of the epoch kernel on this tree (roofline JSON + stall analysis)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/r2z_hogwild python bench.py --no-cpu-baseline --fit 0 --steps 1 --warmup 3 > gpurun_out/ncu_hw.log 2>&1; echo ncu_hw=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fit 0 > /dev/null 2>&1; echo launches=$?
