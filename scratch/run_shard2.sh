timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_comm_nccl.py -x -q > gpurun_out/gpu_shard.log 2>&1; echo "shard rc=$?"; tail -5 gpurun_out/gpu_shard.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
