# round 2: refresh/gather minimum-blocks sweep (128 / 96 / 80 registers)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_RG_MINB=8" "SMCL_RG_MINB=10" "SMCL_RG_MINB=12" "SMCL_RG_MINB=8"; do
  env $v timeout 600 $B > gpurun_out/r02_rgm.json 2> gpurun_out/r02_rgm.err || tail -5 gpurun_out/r02_rgm.err
  python -c "import json; d=json.load(open('gpurun_out/r02_rgm.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','refresh_gather_ms','svgd_ms','total_ms')})"
done
