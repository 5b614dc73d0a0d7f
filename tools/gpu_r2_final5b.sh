# final build, step 2: GPU suite, smoke, default bench (roofline.measured of this build), reference arm
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python bench.py --config c5 --no-cpu-baseline --fit 0 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2=$?
