# round 2: kidnap (bricked HBM table): GN warps per SM
for v in "X=1" "SMCL_FAST_CFG_GN=4x20" "SMCL_FAST_CFG_GN=4x24"; do
env $v timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline --profile-json gpurun_out/r02_kid_prof.json > gpurun_out/r02_kid.json 2> gpurun_out/r02_kid.err
python - <<PY
import json
d=json.load(open('gpurun_out/r02_kid_prof.json'))['stage_profiles']
full=[p for p in d if p['ll_points']>0]
print("$v", {k: round(sum(p[k] for p in full)/len(full),3) for k in ('gn_kernel_ms','ll_kernel_ms','total_ms')})
PY
done
