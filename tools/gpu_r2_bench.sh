# default bench on the final tree (roofline.measured from the committed capture of this build)
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c3b.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/bench_c3b.log
