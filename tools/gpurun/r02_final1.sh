# round 2: default bench (with the CPU baseline), reference arm, kidnap workload, GPU suite
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline > gpurun_out/r02_bench_kidnap.json 2> gpurun_out/r02_bench_kidnap.err; echo "kidnap rc=$?"
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "ref rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests4.log 2>&1; tail -2 gpurun_out/r02_gputests4.log
