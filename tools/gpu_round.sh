# full GPU check: all -m gpu tests, smoke, default bench (with CPU baseline), C4 online bench, launch list
python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
