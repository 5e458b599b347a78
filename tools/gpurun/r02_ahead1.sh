# round 2: GN ahead of the neighbour pass (concurrent K1), configurations
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_GN_AHEAD=0" "X=1" "SMCL_GN_AHEAD_CFG=424" "SMCL_GN_AHEAD_CFG=412" "SMCL_GN_AHEAD_CFG=408"; do
  env $v timeout 600 $B > gpurun_out/r02_a1.json 2> gpurun_out/r02_a1.err || tail -5 gpurun_out/r02_a1.err
  python -c "import json; d=json.load(open('gpurun_out/r02_a1.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','refresh_gather_ms','svgd_ms','total_ms')})"
done
./examples/scenario_callsite
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
