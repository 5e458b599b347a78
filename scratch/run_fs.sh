timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/gpu_fs.log 2>&1; echo "fs rc=$?"; tail -25 gpurun_out/gpu_fs.log
