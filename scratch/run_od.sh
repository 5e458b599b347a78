timeout 900 python -m pytest tests/test_gpu_scenario.py -x -q -s -k outdoor > gpurun_out/gpu_od.log 2>&1; echo "od rc=$?"; grep -E "outdoor|passed|failed|Error" gpurun_out/gpu_od.log | head
