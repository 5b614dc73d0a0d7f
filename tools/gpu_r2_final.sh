# round-2 evidence: full GPU suite + smoke, default bench (+ fit leg, CPU baseline), reference
# arm, C2 / C4 / C5 benches, launch list, ncu --set full of the epoch / hash / explicit / GSM
# kernels, GSM C2/C3, public-API online + fit costs, DSGD stage times, N=2 shared-GPU path
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c3.log 2>&1; echo bench=$?
python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo c2=$?
python bench.py --config c4 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
python bench.py --config c5 --no-cpu-baseline --fit 0 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --fit 0 > /dev/null 2>&1; echo launches=$?
ncu --set full --import-source on --clock-control none -k regex:hogwild_kernel -s 3 -c 1 -o gpurun_out/r2f_hogwild python bench.py --no-cpu-baseline --fit 0 --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu_hw=$?
ncu --set full --import-source on --clock-control none -k regex:hash_count_kernel -c 1 -o gpurun_out/r2f_hash_count python bench.py --no-cpu-baseline --fit 0 --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu_hash=$?
ncu --set full --import-source on --clock-control none -k regex:explicit_row_kernel -c 1 -o gpurun_out/r2f_explicit_row python bench.py --no-cpu-baseline --fit 0 --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu_expl=$?
timeout 900 python tools/bench_gsm.py c2 --sample 8 > gpurun_out/gsm_c2.log 2>&1; echo gsm_c2=$?
timeout 900 python tools/bench_gsm.py c3 --sample 8 > gpurun_out/gsm_c3.log 2>&1; echo gsm_c3=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsm_stats_tc_kernel -c 1 -o gpurun_out/r2f_gsm_tc_c3 python tools/bench_gsm.py c3 --sample 1 > /dev/null 2>&1; echo ncu_gsm=$?
timeout 1200 python tools/api_costs.py fit online > gpurun_out/api_costs.log 2>&1; echo api=$?
timeout 900 python tools/dsgd_stage_time.py > gpurun_out/dsgd_stage.log 2>&1; echo dsgd_stage=$?
CULSH_DIST_BACKEND=gloo CULSH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank_peer.log 2>&1; echo b2=$?
timeout 900 python tools/absorb_breakdown.py > gpurun_out/absorb_breakdown.log 2>&1; echo ab=$?
timeout 600 python tools/lsh_breakdown.py > gpurun_out/lsh_breakdown.log 2>&1; echo lb=$?
