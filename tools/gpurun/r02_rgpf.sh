# round 2: neighbour pass: window-evaluation pose prefetch
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_RG_PF=1" "SMCL_RG_PF=2"; do
  env $v timeout 600 $B > gpurun_out/r02_rgpf.json 2> gpurun_out/r02_rgpf.err || tail -5 gpurun_out/r02_rgpf.err
  python -c "import json; d=json.load(open('gpurun_out/r02_rgpf.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('refresh_gather_ms','total_ms')})"
done
