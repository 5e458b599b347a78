# round 2: smoothing rounds alternate sweep direction (L2 reuse of the list rows)
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py -x -q -m gpu 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_SMOOTH_NOREV=1" "X=1" "SMCL_SMOOTH_NOREV=1"; do
  env $v timeout 600 $B > gpurun_out/r02_smrev.json 2> gpurun_out/r02_smrev.err || tail -5 gpurun_out/r02_smrev.err
  python -c "import json; d=json.load(open('gpurun_out/r02_smrev.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','smooth_ms','bayes_ms','total_ms')})"
done
