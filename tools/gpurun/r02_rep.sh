# round 2: representative argmax partials from the final normalisation sweep
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_rep.json 2> gpurun_out/r02_rep.err || tail -5 gpurun_out/r02_rep.err
python -c "import json; d=json.load(open('gpurun_out/r02_rep.json')); print(round(d['ms_per_step'],3), d['gpu_launches'], {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('bayes_ms','smooth_ms','total_ms')})"
timeout 1200 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_golden.py tests/test_gpu_filter.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance_c2.py tests/test_gpu_scenario.py -x -q 2>&1 | tail -2
