# A/B the working tree against an older tree exported under alt/old (same box, alternating)
for r in 1 2; do
  (cd alt/old && python bench.py --no-cpu-baseline --steps 20 > ../../gpurun_out/ab_old_$r.log 2>&1)
  python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_new_$r.log 2>&1
done
