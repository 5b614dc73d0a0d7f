mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "hash or Hash or lsh or LSH or topk or simlsh or online or Online or scale or dist" > gpurun_out/t_i.log 2>&1; echo t=$?
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --fit 0 --steps 5 > gpurun_out/bench_lsh_$i.log 2>&1; echo bench=$?; done
timeout 600 python tools/lsh_breakdown.py > gpurun_out/lsh_breakdown.log 2>&1; echo lb=$?
