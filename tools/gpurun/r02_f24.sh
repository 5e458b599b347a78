# round 2: K1 queue stores the raw fraction bits (float built in phase B for candidates only)
timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_fullsize.py tests/test_gpu_filter.py -x -q -m gpu 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "X=1"; do
  env $v timeout 600 $B > gpurun_out/r02_f24.json 2> gpurun_out/r02_f24.err || tail -5 gpurun_out/r02_f24.err
  python -c "import json; d=json.load(open('gpurun_out/r02_f24.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','ll_kernel_ms','total_ms')})"
done
