for c in 8x14 4x16 4x20 4x24; do
SMCL_FAST_CFG=$c timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bc_$c.json 2> gpurun_out/bc_$c.err
python -c "import json; d=json.load(open('gpurun_out/bc_$c.json')); s=d['stage_ms']; print('$c', 'ms/step', round(d['ms_per_step'],3), 'gn', round(s['gn_kernel_ms'],3), 'll', round(s['ll_kernel_ms'],3))"
done
