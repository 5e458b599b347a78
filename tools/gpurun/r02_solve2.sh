# round 2: solve rework: failing test detail + guard statistics
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_acceptance_c2.py -x -q 2>&1 | grep -v "^\.\|passed" | head -60
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_solve.json 2> gpurun_out/r02_solve.err || tail -5 gpurun_out/r02_solve.err
python -c "import json; d=json.load(open('gpurun_out/r02_solve.json')); print(round(d['ms_per_step'],3), d['frame_ms'], d['hash_guard'])"
