# round-2 baseline: GPU suite, default bench, and ncu --set full of every hot kernel
# (hash_count, explicit_mask, hogwild epoch, exact column pass)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
ncu --set full --import-source on --clock-control none -k regex:hash_count_kernel -s 1 -c 1 -o gpurun_out/r2_hash_count python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_hash.log 2>&1; echo ncu_hash=$?
ncu --set full --import-source on --clock-control none -k regex:explicit_mask_kernel -c 1 -o gpurun_out/r2_explicit_mask python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_mask.log 2>&1; echo ncu_mask=$?
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/r2_hogwild python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_hw.log 2>&1; echo ncu_hw=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:exact_col_kernel -c 1 -o gpurun_out/r2_exact_col python tools/bench_modes.py c3 --exact-only > gpurun_out/ncu_exact.log 2>&1; echo ncu_exact=$?
