timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('global', d['ms_per_step'], d['stage_ms']['gn_kernel_ms'], d['stage_ms']['ll_kernel_ms'])"
timeout 600 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline > gpurun_out/bench_kid.json 2> gpurun_out/bench_kid.err; echo "kid rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_kid.json')); print('kidnap', d['ms_per_step'], d['stage_ms']['gn_kernel_ms'], d['stage_ms']['ll_kernel_ms'], d['config']['engine_setup_s'])"
