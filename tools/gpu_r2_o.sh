mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "exact or train_full or parallel or online or dsgd or scale or basic or api or golden" > gpurun_out/t_o.log 2>&1; echo t=$?
(cd alt/old && timeout 900 python tools/bench_modes.py c3 --exact-only > ../../gpurun_out/modes_old_u.log 2>&1); echo mo=$?
timeout 900 python tools/bench_modes.py c3 --exact-only > gpurun_out/modes_new_u.log 2>&1; echo mn=$?
(cd alt/old && timeout 1200 python tools/bench_modes.py c3 --exact-only --structured > ../../gpurun_out/modes_old_s.log 2>&1); echo mos=$?
timeout 1200 python tools/bench_modes.py c3 --exact-only --structured > gpurun_out/modes_new_s.log 2>&1; echo mns=$?
