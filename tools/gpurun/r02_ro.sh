# round 2: reorder kernel with a (128, 1) launch bound
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1"; do
  env $v timeout 600 $B > gpurun_out/r02_ro.json 2> gpurun_out/r02_ro.err || tail -5 gpurun_out/r02_ro.err
  python -c "import json; d=json.load(open('gpurun_out/r02_ro.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('reorder_ms','smooth_ms','total_ms')})"
done
