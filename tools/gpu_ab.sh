# A/B the working tree against an older tree exported under alt/old (same box, alternating)
mkdir -p gpurun_out
for r in 1 2; do
  (cd alt/old && python bench.py --no-cpu-baseline --fit 0 --steps 20 > ../../gpurun_out/ab_old_$r.log 2>&1)
  python bench.py --no-cpu-baseline --fit 0 --steps 20 > gpurun_out/ab_new_$r.log 2>&1
done
(cd alt/old && python bench.py --config c5 --no-cpu-baseline --fit 0 --steps 10 > ../../gpurun_out/ab_old_c5.log 2>&1)
python bench.py --config c5 --no-cpu-baseline --fit 0 --steps 10 > gpurun_out/ab_new_c5.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "hogwild or Hogwild" > gpurun_out/ab_tests.log 2>&1; echo tests=$?
