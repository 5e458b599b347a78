# round 2: GN pass concurrent with the refresh/gather kernel (launched after the reorder), K1 configurations
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_GN_AHEAD=0" "X=1" "SMCL_GN_AHEAD_CFG=4x12" "SMCL_GN_AHEAD_CFG=4x8" "SMCL_GN_AHEAD_CFG=4x24"; do
  env $v timeout 600 $B > gpurun_out/r02_a2.json 2> gpurun_out/r02_a2.err || tail -5 gpurun_out/r02_a2.err
  python -c "import json; d=json.load(open('gpurun_out/r02_a2.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','refresh_gather_ms','svgd_ms','total_ms')})"
done
timeout 1500 python -m pytest tests/test_gpu_parity_step.py tests/test_gpu_sharded.py tests/test_gpu_filter.py tests/test_gpu_sharded_mp.py tests/test_gpu_facade.py -x -q 2>&1 | tail -5
