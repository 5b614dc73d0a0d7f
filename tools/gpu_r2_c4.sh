mkdir -p gpurun_out
python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
tail -c 800 gpurun_out/bench_c4.log
