# round 2, call 6: GSM drift-sync A/B with relaxed polling + fit breakdown
mkdir -p gpurun_out
for s in "16,2" "32,2" "32,4" "64,2" "64,4" "128,2"; do
  CULSH_GSM_SYNC=$s timeout 600 python tools/bench_gsm.py c2 --sample 1 > gpurun_out/gsm_c2_$s.log 2>&1; echo c2 $s $?
  CULSH_GSM_SYNC=$s timeout 600 python tools/bench_gsm.py c3 --sample 1 > gpurun_out/gsm_c3_$s.log 2>&1; echo c3 $s $?
done
timeout 900 python tools/fit_breakdown.py > gpurun_out/fit_breakdown.log 2>&1; echo fit=$?
