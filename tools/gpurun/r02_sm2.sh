# round 2: smoothing grid-stride with the next rows prefetched; K2 with 2 points per lane in flight
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_SMOOTH_PF=6" "SMCL_SMOOTH_PF=12" "SMCL_FAST_CFG_LL=L2x83"; do
  env $v timeout 600 $B > gpurun_out/r02_sm2.json 2> gpurun_out/r02_sm2.err || tail -5 gpurun_out/r02_sm2.err
  python -c "import json; d=json.load(open('gpurun_out/r02_sm2.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('ll_kernel_ms','smooth_ms','total_ms')}, d['frame_ms'])"
done
