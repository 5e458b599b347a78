# round 2: SVGD neighbour prefetch through cp.async shared-memory slots
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_SVGD_CFG=3" "SMCL_SVGD_CFG=42" "SMCL_SVGD_CFG=43" "SMCL_SVGD_CFG=52"; do
  env $v timeout 600 $B > gpurun_out/r02_svgd3.json 2> gpurun_out/r02_svgd3.err || tail -5 gpurun_out/r02_svgd3.err
  python -c "import json; d=json.load(open('gpurun_out/r02_svgd3.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('svgd_ms','total_ms')})"
done
SMCL_SVGD_CFG=43 timeout 600 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py -x -q 2>&1 | tail -2
