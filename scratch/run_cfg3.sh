for c in 4x22 4x24 4x20; do
  SMCL_FAST_CFG_GN=$c timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_c.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_c.json').read().strip().splitlines()[-1])
print('cfg $c', round(d['ms_per_step'],3), round(d['stage_ms']['gn_kernel_ms'],3))"
done
