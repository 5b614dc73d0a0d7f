# round-2 baseline: GPU suite, smoke, default bench, launch list and ncu --set full of every
# hot kernel (hash_count, explicit_mask, hogwild epoch, exact column pass) + SASS summary
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none -k regex:hash_count_kernel -c 1 -o gpurun_out/r2_hash_count python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_hash.log 2>&1; echo ncu_hash=$?
ncu --set full --import-source on --clock-control none -k regex:explicit_mask_kernel -c 1 -o gpurun_out/r2_explicit_mask python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_mask.log 2>&1; echo ncu_mask=$?
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/r2_hogwild python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_hw.log 2>&1; echo ncu_hw=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:exact_col_kernel -c 1 -o gpurun_out/r2_exact_col python tools/bench_modes.py c3 --exact-only > gpurun_out/ncu_exact.log 2>&1; echo ncu_exact=$?
