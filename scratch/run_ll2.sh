timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for c in 4x24 L8x8 L4x8 L8x4; do
SMCL_FAST_CFG=$c timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bl_$c.json 2> gpurun_out/bl_$c.err
python -c "import json; d=json.load(open('gpurun_out/bl_$c.json')); s=d['stage_ms']; print('$c', 'ms/step', round(d['ms_per_step'],3), 'gn', round(s['gn_kernel_ms'],3), 'll', round(s['ll_kernel_ms'],3))"
done
