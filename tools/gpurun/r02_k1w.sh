# round 2: K1 rotation re-read from shared memory per phase-B batch (80 registers): 24 warps per SM
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_FAST_CFG_GN=4x20"; do
  env $v timeout 600 $B > gpurun_out/r02_k1w.json 2> gpurun_out/r02_k1w.err || tail -5 gpurun_out/r02_k1w.err
  python -c "import json; d=json.load(open('gpurun_out/r02_k1w.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','ll_kernel_ms','smooth_ms','total_ms')})"
done
timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py tests/test_gpu_fullsize.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
