# round 2: sharded engines (asynchronous migration counts), profile accounting, two-process test
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_sharded_mp.py tests/test_gpu_comm_nccl.py -x -q 2>&1 | tail -4
