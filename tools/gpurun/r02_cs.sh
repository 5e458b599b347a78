# round 2: chunk-serial sums staged by 256 threads; host gap diagnostic
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_cs.json 2> gpurun_out/r02_cs.err || tail -5 gpurun_out/r02_cs.err
python -c "import json; d=json.load(open('gpurun_out/r02_cs.json')); print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()})"
timeout 300 python tools/diag_host_gap.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_golden.py tests/test_gpu_filter.py -x -q 2>&1 | tail -3
