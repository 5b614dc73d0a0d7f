# round-2 final evidence on the final tree (after the exact RMSE sum)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/r2g_hogwild python bench.py --no-cpu-baseline --fit 0 --steps 1 --warmup 3 > gpurun_out/ncu_hw.log 2>&1; echo ncu_hw=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fit 0 > /dev/null 2>&1; echo launches=$?
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2=$?
python bench.py --config c5 --no-cpu-baseline --fit 0 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 900 python tools/api_costs.py fit exact > gpurun_out/api_costs.log 2>&1; echo api=$?; tail -3 gpurun_out/api_costs.log
timeout 600 python tools/rmse_phases.py > gpurun_out/rmse_phases.log 2>&1; echo rp=$?; tail -3 gpurun_out/rmse_phases.log
