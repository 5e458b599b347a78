for v in 0 10 12; do
SMCL_RG_MINB=$v timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/rgm_$v.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/rgm_$v.json')); print('$v', d['ms_per_step'], d['stage_ms']['refresh_gather_ms'])"
done
