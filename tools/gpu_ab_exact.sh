# A/B of the exact (bit-identical) modes: full GPU suite, then bench_modes (uniform x2,
# structured) and the C4 online bench for alt/old and the working tree
python -m pytest tests -m gpu -x -q > gpurun_out/t_ex.log 2>&1; echo t=$?
for r in 1 2; do
 (cd alt/old && python tools/bench_modes.py c3 --exact-only > ../../gpurun_out/ex_old_u_$r.log 2>&1)
 python tools/bench_modes.py c3 --exact-only > gpurun_out/ex_new_u_$r.log 2>&1
done
(cd alt/old && python tools/bench_modes.py c3 --structured --exact-only > ../../gpurun_out/ex_old_s.log 2>&1)
python tools/bench_modes.py c3 --structured --exact-only > gpurun_out/ex_new_s.log 2>&1
(cd alt/old && python bench.py --config c4 > ../../gpurun_out/ex_old_c4.log 2>&1)
python bench.py --config c4 > gpurun_out/ex_new_c4.log 2>&1
