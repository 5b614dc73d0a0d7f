# one ncu --set full capture of the Hogwild epoch kernel (bench C3 config)
ncu --set full --import-source on --clock-control none -k regex:hogwild -s 3 -c 1 -o gpurun_out/prof_cur python bench.py --no-cpu-baseline --steps 1 --warmup 3 "$@" > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
