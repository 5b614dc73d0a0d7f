# round 2, call 7: full GPU suite, GSM default, D2H strategies, compute-sanitizer
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 600 python tools/bench_gsm.py c3 --sample 4 > gpurun_out/gsm_c3.log 2>&1; echo gsm_c3=$?
timeout 600 python tools/bench_gsm.py c2 --sample 4 > gpurun_out/gsm_c2.log 2>&1; echo gsm_c2=$?
timeout 600 python tools/d2h_bench.py > gpurun_out/d2h.log 2>&1; echo d2h=$?
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_kernels.py all > gpurun_out/san_memcheck.log 2>&1; echo memcheck=$?
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 50 python tools/sanitize_kernels.py deterministic > gpurun_out/san_racecheck.log 2>&1; echo racecheck=$?
timeout 1200 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_kernels.py deterministic > gpurun_out/san_synccheck.log 2>&1; echo synccheck=$?
