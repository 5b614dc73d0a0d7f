mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "online or absorb or increment or c4 or extend or exact or train_full" > gpurun_out/t_r.log 2>&1; echo t=$?
for r in 1 2; do
  (cd alt/old && timeout 900 python bench.py --config c4 > ../../gpurun_out/c4_old_$r.log 2>&1)
  timeout 900 python bench.py --config c4 > gpurun_out/c4_new_$r.log 2>&1
done
echo done
