for v in "X=1" "SMCL_FAST_CFG_LL=4x24" "SMCL_FAST_CFG_LL=4x16" "SMCL_FAST_CFG_LL=8x14"; do
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_b9.json 2> gpurun_out/r02_b9.err
  python -c "import json; d=json.load(open('gpurun_out/r02_b9.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','ll_kernel_ms')})"
done
