for v in 0 5 6 8; do
SMCL_SVGD_MINB=$v timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bs_$v.json 2> gpurun_out/bs_$v.err
python -c "import json; d=json.load(open('gpurun_out/bs_$v.json')); s=d['stage_ms']; print('$v', 'ms/step', round(d['ms_per_step'],3), 'svgd', round(s['svgd_ms'],3))"
done
