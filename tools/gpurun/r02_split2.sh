# round 2: gate split threshold margin sweep
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_LL_SPLIT_MARGIN=-32" "SMCL_LL_SPLIT_MARGIN=0" "SMCL_LL_SPLIT_MARGIN=16" "SMCL_LL_SPLIT_MARGIN=48"; do
  env $v timeout 600 $B > gpurun_out/r02_split.json 2> gpurun_out/r02_split.err || tail -5 gpurun_out/r02_split.err
  python -c "import json; d=json.load(open('gpurun_out/r02_split.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('ll_kernel_ms','total_ms')})"
done
