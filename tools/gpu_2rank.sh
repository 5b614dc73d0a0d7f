# the N = 2 bench path end to end on the final tree (both ranks share the one GPU: not a scaling number)
mkdir -p gpurun_out
CULSH_DIST_BACKEND=gloo CULSH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2rank_peer.log 2>&1; echo b2=$?
tail -c 1500 gpurun_out/bench_2rank_peer.log
