timeout 900 python -m pytest tests/test_gpu_scan_prep.py tests/test_gpu_map.py -x -q > gpurun_out/gpu_scan.log 2>&1; echo "scan rc=$?"; tail -30 gpurun_out/gpu_scan.log
