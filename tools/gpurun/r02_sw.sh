# round 2: smoothing with the neighbour-index window staged in shared memory
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_SMOOTH_WIN=0" "SMCL_SMOOTH_WIN=512" "SMCL_SMOOTH_WIN=1024" "SMCL_SMOOTH_WIN=2048"; do
  env $v timeout 600 $B > gpurun_out/r02_sw.json 2> gpurun_out/r02_sw.err || tail -5 gpurun_out/r02_sw.err
  python -c "import json; d=json.load(open('gpurun_out/r02_sw.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','ll_kernel_ms','smooth_ms','total_ms')})"
done
timeout 900 python -m pytest tests/test_gpu_parity_step.py tests/test_gpu_stages.py tests/test_gpu_golden.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -3
