# round 2: likelihood pass with / without the K2a gate
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_NO_LL_GATE=1"; do
  env $v timeout 600 $B > gpurun_out/r02_gate.json 2> gpurun_out/r02_gate.err || tail -5 gpurun_out/r02_gate.err
  python -c "import json; d=json.load(open('gpurun_out/r02_gate.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('ll_kernel_ms','total_ms')})"
done
