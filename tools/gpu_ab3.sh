# A/B of the working tree against HEAD exported under alt/old (same box, alternating), then the GPU suite
mkdir -p gpurun_out
for r in 1 2 3; do
  (cd alt/old && python bench.py --no-cpu-baseline --fit 0 --steps 20 > ../../gpurun_out/ab_old_$r.log 2>&1)
  python bench.py --no-cpu-baseline --fit 0 --steps 20 > gpurun_out/ab_new_$r.log 2>&1
done
(cd alt/old && python bench.py --config c5 --no-cpu-baseline --fit 0 --steps 10 > ../../gpurun_out/ab_old_c5.log 2>&1)
python bench.py --config c5 --no-cpu-baseline --fit 0 --steps 10 > gpurun_out/ab_new_c5.log 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    l=[x for x in open(f) if x.startswith('{')]
    if l:
        d=json.loads(l[-1]); print(f, round(d['ms_per_step'],3), d.get('e2e',{}).get('value'), d.get('clocks',{}).get('sm_mhz'))
    else: print(f, 'no line')
PY
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ab_tests.log
