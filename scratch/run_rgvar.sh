for v in 0 10 12 16; do
SMCL_RG_MINB=$v timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_$v.json 2> gpurun_out/b_$v.err
python -c "import json; d=json.load(open('gpurun_out/b_$v.json')); print('$v', 'ms/step', round(d['ms_per_step'],3), 'rg', round(d['stage_ms']['refresh_gather_ms'],3))"
done
