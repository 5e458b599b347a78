timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/gpu_shard.log 2>&1; echo "shard rc=$?"; tail -15 gpurun_out/gpu_shard.log
