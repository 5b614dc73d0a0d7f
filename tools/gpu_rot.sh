python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "Packed" > gpurun_out/t_rot.log 2>&1; echo tests=$?
python bench.py --no-cpu-baseline --rotate 1 > gpurun_out/b_rot1.log 2>&1; echo b1=$?
python bench.py --no-cpu-baseline --rotate 0 > gpurun_out/b_rot0.log 2>&1; echo b0=$?
python tools/debug_c3_structured.py c3 > gpurun_out/dbg.log 2>&1; echo dbg=$?
