# round 2: GN pass matched count folded into the solve
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_sc.json 2> gpurun_out/r02_sc.err || tail -5 gpurun_out/r02_sc.err
python -c "import json; d=json.load(open('gpurun_out/r02_sc.json')); print(round(d['ms_per_step'],3), d['gpu_launches'], d['roofline']['algorithmic_bytes_per_launch'], {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('solve_ms','total_ms')})"
timeout 1500 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_sharded.py tests/test_gpu_likelihood.py -x -q 2>&1 | tail -2
