./build/tools/ffma2_micro > gpurun_out/ffma2.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity_step.py tests/test_gpu_acceptance_c2.py -x -q -s > gpurun_out/r02_parity1.log 2>&1; echo "tests rc=$?"
