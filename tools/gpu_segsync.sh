# work-segment merge A/B on skewed data: averaged (1/S at the end) vs shared every 32 updates
mkdir -p gpurun_out
CAPS=2,1,0.5 CULSH_SEGMENT_SYNC=0 timeout 600 python tools/skew_cap_sweep.py 8 c2 > gpurun_out/seg_avg_c2.json 2>gpurun_out/seg_avg_c2.err; echo avg_c2=$?
CAPS=2,1,0.5 CULSH_SEGMENT_SYNC=1 timeout 600 python tools/skew_cap_sweep.py 8 c2 > gpurun_out/seg_sync_c2.json 2>gpurun_out/seg_sync_c2.err; echo sync_c2=$?
CAPS=2,1,0.5 CULSH_SEGMENT_SYNC=0 timeout 900 python tools/skew_cap_sweep.py 6 c3 > gpurun_out/seg_avg_c3.json 2>gpurun_out/seg_avg_c3.err; echo avg_c3=$?
CAPS=2,1,0.5 CULSH_SEGMENT_SYNC=1 timeout 900 python tools/skew_cap_sweep.py 6 c3 > gpurun_out/seg_sync_c3.json 2>gpurun_out/seg_sync_c3.err; echo sync_c3=$?
cat gpurun_out/seg_*.json
