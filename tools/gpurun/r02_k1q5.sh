# round 2: queue K1: rotation loaded once per step
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_K1_QUEUE=2x28"; do
  env $v timeout 600 $B > gpurun_out/r02_k1q5.json 2> gpurun_out/r02_k1q5.err || tail -5 gpurun_out/r02_k1q5.err
  python -c "import json; d=json.load(open('gpurun_out/r02_k1q5.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','total_ms')})"
done
