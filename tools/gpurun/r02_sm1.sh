# round 2: lean fast-path solve; smoothing with a persisting L2 window on the kval rows
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_SMOOTH_L2=1.0" "SMCL_SMOOTH_L2=0.6"; do
  env $v timeout 600 $B > gpurun_out/r02_sm1.json 2> gpurun_out/r02_sm1.err || tail -5 gpurun_out/r02_sm1.err
  grep smooth-l2 gpurun_out/r02_sm1.err | head -1
  python -c "import json; d=json.load(open('gpurun_out/r02_sm1.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('solve_ms','smooth_ms','total_ms')})"
done
timeout 900 python -m pytest tests/test_gpu_parity_step.py tests/test_gpu_stages.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3
