# round 2: smoothing register budget (CTAs per SM)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_SMOOTH_MINB=12" "SMCL_SMOOTH_MINB=1" "SMCL_SMOOTH_MINB=10"; do
  env $v timeout 600 $B > gpurun_out/r02_smb.json 2> gpurun_out/r02_smb.err || tail -5 gpurun_out/r02_smb.err
  python -c "import json; d=json.load(open('gpurun_out/r02_smb.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('smooth_ms','total_ms')})"
done
