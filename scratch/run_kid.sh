timeout 600 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline > gpurun_out/bench_kid.json 2> gpurun_out/bench_kid.err; echo "kid rc=$?"; tail -3 gpurun_out/bench_kid.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_kid.json'))
print('ms/step', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['ms_per_step'], 'setup', d['config']['engine_setup_s'])
print({k: round(v,3) for k,v in d['stage_ms'].items()})
print(d['e2e_raw_points']['ms_per_step'], d['scan_prep_ms'])
PY
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('global ms/step', d['ms_per_step'], d['value'], d['e2e']['value'])"
