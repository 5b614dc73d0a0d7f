mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "hogwild or Hogwild or work or dsgd or dist or Packed or packed" > gpurun_out/t_h.log 2>&1; echo t=$?
timeout 900 python tools/dsgd_stage_time.py > gpurun_out/dsgd_stage.log 2>&1; echo dsgd=$?
timeout 900 python bench.py --no-cpu-baseline --fit 0 --steps 10 > gpurun_out/bench_c3_check.log 2>&1; echo bench=$?
