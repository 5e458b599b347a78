timeout 1200 python -m pytest tests/test_gpu_scenario.py -x -q -s > gpurun_out/gpu_scen.log 2>&1; echo "scen rc=$?"; grep -E "C6|C7|passed|failed|Error|assert" gpurun_out/gpu_scen.log | head -20
