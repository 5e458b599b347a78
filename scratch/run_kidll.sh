for c in L8x8 4x24 4x16 8x14; do
SMCL_FAST_CFG_LL=$c timeout 600 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline > gpurun_out/bk_$c.json 2> gpurun_out/bk_$c.err
python -c "import json; d=json.load(open('gpurun_out/bk_$c.json')); print('$c', d['ms_per_step'], d['stage_ms']['gn_kernel_ms'], d['stage_ms']['ll_kernel_ms'])"
done
SMCL_FAST_CFG_LL=4x24 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bg.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bg.json')); print('global 4x24', d['ms_per_step'], d['stage_ms']['ll_kernel_ms'])"
