# round-end evidence: full GPU suite, smoke, default bench (+CPU baseline), reference arm,
# C4 online bench, launch list, one ncu --set full capture of the epoch kernel, C5 bench,
# DSGD per-GPU stage times, and the N = 2 bench path with ranks sharing the GPU over gloo
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/prof_hw14 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
python bench.py --config c5 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
python tools/dsgd_stage_time.py > gpurun_out/dsgd_stage.log 2>&1; echo dsgd_stage=$?
CULSH_DIST_BACKEND=gloo CULSH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_2rank_gloo.log 2>&1; echo b2=$?
