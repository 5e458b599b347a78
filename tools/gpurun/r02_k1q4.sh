# round 2: queue K1 warps per SM after the enqueue rework
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "SMCL_K1_QUEUE=4x18" "SMCL_K1_QUEUE=2x24" "SMCL_K1_QUEUE=2x28" "SMCL_K1_QUEUE=4x16"; do
  env $v timeout 600 $B > gpurun_out/r02_k1q4.json 2> gpurun_out/r02_k1q4.err || tail -5 gpurun_out/r02_k1q4.err
  python -c "import json; d=json.load(open('gpurun_out/r02_k1q4.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','total_ms')})"
done
