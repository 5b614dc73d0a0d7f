# compute-sanitizer is closed on the pool: run the cases plainly (each is checked against the oracle)
mkdir -p gpurun_out
timeout 600 python tools/sanitize_kernels.py all > gpurun_out/san_cases.log 2>&1; echo cases=$?; tail -3 gpurun_out/san_cases.log
