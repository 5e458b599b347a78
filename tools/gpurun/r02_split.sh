# round 2: speculative likelihood-gate split from the GN pass's counts
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_NO_LL_SPLIT=1"; do
  env $v timeout 600 $B > gpurun_out/r02_split.json 2> gpurun_out/r02_split.err || tail -5 gpurun_out/r02_split.err
  python -c "import json; d=json.load(open('gpurun_out/r02_split.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('ll_kernel_ms','total_ms')})"
done
timeout 1500 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py tests/test_gpu_scenario.py tests/test_gpu_acceptance_c2.py -x -q 2>&1 | tail -2
