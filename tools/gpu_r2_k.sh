mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/t_k.log 2>&1; echo t=$?
CULSH_DIST_BACKEND=gloo CULSH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank_auto.log 2>&1; echo b2=$?
