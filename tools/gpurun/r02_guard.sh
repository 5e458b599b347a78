# round 2: host LSH guard checks only the flagged particles; solve on the packed lower triangle
timeout 900 python -m pytest tests/test_gpu_lsh_fixtures.py tests/test_gpu_stages.py tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_acceptance_c2.py tests/test_gpu_sharded.py -x -q 2>&1 | grep -v "^\.\+ *\[" | tail -30
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_guard.json 2> gpurun_out/r02_guard.err || tail -5 gpurun_out/r02_guard.err
python -c "import json; d=json.load(open('gpurun_out/r02_guard.json')); print(round(d['ms_per_step'],3), d['frame_ms']['full_scan'], d['hash_guard'], {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('solve_ms','total_ms')})"
