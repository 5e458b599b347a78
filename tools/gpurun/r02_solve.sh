# round 2: solve on the packed lower triangle, fast path with pivot reciprocals
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1"; do
  env $v timeout 600 $B > gpurun_out/r02_solve.json 2> gpurun_out/r02_solve.err || tail -5 gpurun_out/r02_solve.err
  python -c "import json; d=json.load(open('gpurun_out/r02_solve.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('solve_ms','gn_kernel_ms','ll_kernel_ms','total_ms')})"
done
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_acceptance_c2.py -x -q 2>&1 | tail -2
