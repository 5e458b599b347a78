timeout 900 python -m pytest tests/test_gpu_lsh_fixtures.py -x -q -s > gpurun_out/r02_lshfix.log 2>&1; echo "lshfix rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests.log 2>&1; echo "gpu tests rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
