# round 2: the likelihood pass's profiling match count reuses the Bayes count (unsharded)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_mc.json 2> gpurun_out/r02_mc.err || tail -5 gpurun_out/r02_mc.err
python -c "import json; d=json.load(open('gpurun_out/r02_mc.json')); print(round(d['ms_per_step'],3), d['gpu_launches'], d['roofline']['algorithmic_bytes_per_launch'], {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('bayes_ms','total_ms')})"
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_filter.py tests/test_gpu_stages.py -x -q 2>&1 | tail -2
