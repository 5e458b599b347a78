timeout 600 python bench.py $BENCH_ARGS > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench.json'))
print('ms/step', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'raw', d.get('e2e_raw_points'), d.get('scan_prep_ms'))
print({k: round(v,3) for k,v in d['stage_ms'].items()})
print(d.get('cpu_baseline'))
PY
