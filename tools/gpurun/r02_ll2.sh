# round 2: K2 points in flight per lane
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_FAST_CFG_LL=L2x83" "SMCL_FAST_CFG_LL=L3x83" "SMCL_FAST_CFG_LL=L4x83" "SMCL_FAST_CFG_LL=L2x82"; do
  env $v timeout 600 $B > gpurun_out/r02_ll2.json 2> gpurun_out/r02_ll2.err || tail -5 gpurun_out/r02_ll2.err
  python -c "import json; d=json.load(open('gpurun_out/r02_ll2.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('ll_kernel_ms','total_ms')})"
done
