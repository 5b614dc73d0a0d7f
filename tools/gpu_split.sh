python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "Packed or Hogwild" > gpurun_out/t_split.log 2>&1; echo tests=$?
python bench.py --no-cpu-baseline > gpurun_out/b_quick.log 2>&1; echo bench=$?
python tools/debug_c3_structured.py c3 > gpurun_out/dbg.log 2>&1; echo dbg=$?
