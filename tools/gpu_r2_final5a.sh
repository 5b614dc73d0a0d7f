# final build, step 1: the epoch-kernel capture (roofline JSON) + launch list + the wide-shape tests
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_wide_k.py -q > gpurun_out/widek.log 2>&1; echo widek=$?; tail -3 gpurun_out/widek.log
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/r2h_hogwild python bench.py --no-cpu-baseline --fit 0 --steps 1 --warmup 3 > gpurun_out/ncu_hw.log 2>&1; echo ncu_hw=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fit 0 > /dev/null 2>&1; echo launches=$?
