timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_fullsize.py tests/test_gpu_filter.py tests/test_gpu_golden.py -x -q > gpurun_out/r02_t4.log 2>&1; echo "tests rc=$?"
