# round 2: SVGD prefetch at 3 vs 4 CTAs per SM; host timing around the step
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_SVGD_CFG=4" "SMCL_SVGD_CFG=3"; do
  env $v timeout 600 $B > gpurun_out/r02_svgd.json 2> gpurun_out/r02_svgd.err || tail -5 gpurun_out/r02_svgd.err
  python -c "import json; d=json.load(open('gpurun_out/r02_svgd.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('svgd_ms','total_ms')})"
done
SMCL_HOST_TIMING=1 timeout 300 python tools/diag_host_gap.py > gpurun_out/r02_hostgap.log 2>&1; grep -v "^\[host\]" gpurun_out/r02_hostgap.log | tail -5; grep "^\[host\]" gpurun_out/r02_hostgap.log | tail -4
