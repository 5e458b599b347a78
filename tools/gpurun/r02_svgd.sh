# round 2: SVGD with the next neighbour's pose/step prefetched; host-gap diagnostic
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_SVGD_CFG=0" "SMCL_SVGD_CFG=4" "SMCL_SVGD_CFG=5" "SMCL_SVGD_CFG=6"; do
  env $v timeout 600 $B > gpurun_out/r02_svgd.json 2> gpurun_out/r02_svgd.err || tail -5 gpurun_out/r02_svgd.err
  python -c "import json; d=json.load(open('gpurun_out/r02_svgd.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('svgd_ms','total_ms')})"
done
timeout 300 python tools/diag_host_gap.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
