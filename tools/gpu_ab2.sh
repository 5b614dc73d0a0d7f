# A/B a bench flag on the same box: "$@" = the flag under test (e.g. --rotate 1), 2 rounds alternating
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "Packed or Hogwild" > gpurun_out/t_ab.log 2>&1; echo tests=$?
for r in 1 2; do
  python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_old_$r.log 2>&1
  python bench.py --no-cpu-baseline --steps 20 "$@" > gpurun_out/ab_new_$r.log 2>&1
done
