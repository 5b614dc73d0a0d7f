# A/B of hash_count_kernel variants: alt/<name> trees vs the working tree (tools/lsh_breakdown.py)
for r in 1 2; do
  for d in alt/*/; do v=$(basename $d); echo "$v $r"; (cd alt/$v && python tools/lsh_breakdown.py 2>&1 | grep -E "gpu_span|hash_count"); done
  echo "base $r"; python tools/lsh_breakdown.py 2>&1 | grep -E "gpu_span|hash_count"
done
