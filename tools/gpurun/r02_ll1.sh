# round 2: K2a centered-fraction margin test; K2 with 2 CTAs (16 warps, no spills)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_FAST_CFG_LL=L1x82"; do
  env $v timeout 600 $B > gpurun_out/r02_ll1.json 2> gpurun_out/r02_ll1.err || tail -5 gpurun_out/r02_ll1.err
  python -c "import json; d=json.load(open('gpurun_out/r02_ll1.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','refresh_gather_ms','ll_kernel_ms','total_ms')})"
done
timeout 900 python -m pytest tests/test_gpu_parity_step.py tests/test_gpu_likelihood.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
