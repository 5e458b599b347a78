# round 2: kidnap (bricked table): queue K1 vs staged K1
for v in "X=1" "SMCL_K1_QUEUE_BRICK=1 SMCL_K1_QUEUE=4x16" "SMCL_K1_QUEUE_BRICK=1 SMCL_K1_QUEUE=4x20"; do
env $v timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline --profile-json gpurun_out/r02_kid_prof.json > gpurun_out/r02_kid.json 2> gpurun_out/r02_kid.err
python - <<PY
import json
d=json.load(open('gpurun_out/r02_kid_prof.json'))['stage_profiles']
full=[p for p in d if p['ll_points']>0]
print("$v", {k: round(sum(p[k] for p in full)/len(full),3) for k in ('gn_kernel_ms','ll_kernel_ms','total_ms')})
PY
done
