timeout 900 python -m pytest tests/test_gpu_golden.py -x -q > gpurun_out/gpu_gold.log 2>&1; echo "gold rc=$?"; tail -25 gpurun_out/gpu_gold.log
