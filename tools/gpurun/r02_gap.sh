# round 2: host time between steps after the lazy stage-time reads
SMCL_HOST_TIMING=1 timeout 300 python tools/diag_host_gap.py > gpurun_out/r02_hostgap2.log 2>&1; grep -v "^\[host\]" gpurun_out/r02_hostgap2.log | tail -5; grep "^\[host\]" gpurun_out/r02_hostgap2.log | tail -3
