# round 2: K1 phase-B two-candidate variant at 16 / 20 warps
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_K1_ILP=2" "SMCL_K1_ILP=2 SMCL_FAST_CFG_GN=4x16" "SMCL_FAST_CFG_GN=4x16"; do
  env $v timeout 600 $B > gpurun_out/r02_k1.json 2> gpurun_out/r02_k1.err || tail -5 gpurun_out/r02_k1.err
  python -c "import json; d=json.load(open('gpurun_out/r02_k1.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','refresh_gather_ms','svgd_ms','total_ms')})"
done
