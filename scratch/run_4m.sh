for c in 4x24 4x16 8x14; do
SMCL_FAST_CFG_LL=$c timeout 600 python bench.py --particles 4194304 --scan-points 1024 --steps 3 --no-cpu-baseline > gpurun_out/b4_$c.json 2> /dev/null
python -c "import json; d=json.load(open('gpurun_out/b4_$c.json')); print('$c', d['ms_per_step'], d['stage_ms']['ll_kernel_ms'])"
done
