mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gsm or similarity or pearson" > gpurun_out/t_q.log 2>&1; echo t=$?
timeout 600 python tools/gsm_phases.py c3 4 > gpurun_out/gsmp_c3.log 2>&1; echo p=$?
timeout 600 python tools/bench_gsm.py c3 --sample 8 > gpurun_out/gsm_c3.log 2>&1; echo g3=$?
timeout 600 python tools/bench_gsm.py c2 --sample 8 > gpurun_out/gsm_c2.log 2>&1; echo g2=$?
