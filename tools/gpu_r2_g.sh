mkdir -p gpurun_out
for s in "128,2" "256,4" "512,4" "256,8" "128,4" "64,8"; do
  CULSH_GSM_SYNC=$s timeout 600 python tools/gsm_phases.py c3 6 > gpurun_out/gsmq_c3_$s.log 2>&1; echo $s $?
done
timeout 900 python tools/occupancy_probe.py > gpurun_out/occupancy.log 2>&1; echo occ=$?
