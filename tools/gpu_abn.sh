# A/B/n: every tree under alt/<name> and the working tree, alternating on the same box
for r in 1 2; do
  for d in alt/*/; do
    n=$(basename "$d")
    (cd "$d" && python bench.py --no-cpu-baseline --steps 20 > ../../gpurun_out/ab_${n}_$r.log 2>&1)
  done
  python bench.py --no-cpu-baseline --steps 20 > gpurun_out/ab_new_$r.log 2>&1
done
