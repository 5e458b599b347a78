# round 2: batched window filter; GN pass launched right before the refresh/gather kernel
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_GN_AHEAD=0" "SMCL_GN_AHEAD_CFG=4x16" "SMCL_GN_AHEAD_CFG=4x12" "SMCL_GN_AHEAD_CFG=4x20"; do
  env $v SMCL_STEP_TIMELINE=1 timeout 600 $B > gpurun_out/r02_a5.json 2> gpurun_out/r02_a5.err || tail -5 gpurun_out/r02_a5.err
  python -c "import json; d=json.load(open('gpurun_out/r02_a5.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','refresh_gather_ms','svgd_ms','total_ms')})"
  grep timeline gpurun_out/r02_a5.err | sed -n 8p
done
timeout 900 python -m pytest tests/test_gpu_parity_step.py tests/test_gpu_stages.py tests/test_gpu_lsh_fixtures.py -x -q 2>&1 | tail -3
