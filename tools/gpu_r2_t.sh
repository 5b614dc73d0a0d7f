mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo bench=$?
