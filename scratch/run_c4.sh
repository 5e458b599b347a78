timeout 900 python -m pytest tests/test_gpu_scenario.py -x -q -s -k c4 > gpurun_out/gpu_c4.log 2>&1; echo "c4 rc=$?"; tail -6 gpurun_out/gpu_c4.log
