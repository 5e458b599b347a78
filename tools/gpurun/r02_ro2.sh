# round 2: inverse permutation in the members sweep, pose mirror written by the reorder
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_ro2.json 2> gpurun_out/r02_ro2.err || tail -5 gpurun_out/r02_ro2.err
python -c "import json; d=json.load(open('gpurun_out/r02_ro2.json')); print(round(d['ms_per_step'],3), d['gpu_launches'], {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('sort_ms','reorder_ms','segments_ms','refresh_gather_ms','total_ms')})"
timeout 1500 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_golden.py tests/test_gpu_filter.py tests/test_gpu_sharded.py tests/test_gpu_sharded_mp.py tests/test_gpu_lsh_fixtures.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
