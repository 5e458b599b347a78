# round 2: smoothing rounds chained by programmatic dependent launch
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_sharded.py tests/test_gpu_sharded_mp.py -x -q -m gpu 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_SMOOTH_NOPDL=1" "X=1" "SMCL_SMOOTH_NOPDL=1"; do
  env $v timeout 600 $B > gpurun_out/r02_smpdl.json 2> gpurun_out/r02_smpdl.err || tail -5 gpurun_out/r02_smpdl.err
  python -c "import json; d=json.load(open('gpurun_out/r02_smpdl.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','smooth_ms','bayes_ms','total_ms')})"
done
