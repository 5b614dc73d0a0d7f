mkdir -p gpurun_out
CULSH_GSM_DEBUG=1 timeout 600 python tools/gsm_phases.py c3 8 > gpurun_out/gsmp_c3.log 2>&1; echo p=$?
CULSH_GSM_DEBUG=1 CULSH_GSM_SYNC=0,0 timeout 600 python tools/gsm_phases.py c3 5 > gpurun_out/gsmp_c3_nosync.log 2>&1; echo p=$?
CULSH_GSM_DEBUG=1 CULSH_GSM_SYNC=256,4 timeout 600 python tools/gsm_phases.py c3 6 > gpurun_out/gsmp_c3_256_4.log 2>&1; echo p=$?
