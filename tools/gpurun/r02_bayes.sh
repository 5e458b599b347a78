# round 2: Bayes match counts in the gate's sweep, numerator in the normalisation's argmax sweep
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/r02_bayes.json 2> gpurun_out/r02_bayes.err || tail -5 gpurun_out/r02_bayes.err
python -c "import json; d=json.load(open('gpurun_out/r02_bayes.json')); print(round(d['ms_per_step'],3), d['gpu_launches'], {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('ll_kernel_ms','bayes_ms','smooth_ms','total_ms')})"
timeout 1500 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_golden.py tests/test_gpu_filter.py tests/test_gpu_sharded.py tests/test_gpu_sharded_mp.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance_c2.py tests/test_gpu_scenario.py tests/test_gpu_bench_multirank.py -x -q 2>&1 | tail -2
