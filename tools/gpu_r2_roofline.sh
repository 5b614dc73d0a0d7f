# the epoch kernel's ncu --set full capture of THIS tree (profiles/ncu_roofline_c3.json is
# regenerated from it on the build host, keyed by the tree's source identity)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/r2z_hogwild python bench.py --no-cpu-baseline --fit 0 --steps 1 --warmup 3 > gpurun_out/ncu_hw.log 2>&1; echo ncu_hw=$?
python bench.py --no-cpu-baseline --fit 0 --steps 10 > gpurun_out/bench_check.log 2>&1; echo b=$?
