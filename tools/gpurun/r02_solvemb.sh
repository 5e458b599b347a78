# round 2: solve kernel register budget
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_SOLVE_MINB=4" "SMCL_SOLVE_MINB=6"; do
  env $v timeout 600 $B > gpurun_out/r02_smb2.json 2> gpurun_out/r02_smb2.err || tail -5 gpurun_out/r02_smb2.err
  python -c "import json; d=json.load(open('gpurun_out/r02_smb2.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('solve_ms','total_ms')})"
done
