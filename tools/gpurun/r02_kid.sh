# round 2: kidnap workload stage breakdown of the full-scan frames
timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline --profile-json gpurun_out/r02_kid_prof.json > gpurun_out/r02_kid.json 2> gpurun_out/r02_kid.err; echo "rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02_kid_prof.json'))['stage_profiles']
full=[p for p in d if p['ll_points']>0]
keys=[k for k in full[0] if k.endswith('_ms')]
print(len(full), {k: round(sum(p[k] for p in full)/len(full),3) for k in keys})
PY
