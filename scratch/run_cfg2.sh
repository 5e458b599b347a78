for c in 4x24 4x28 4x32; do
  SMCL_FAST_CFG_GN=$c timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_c$c.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1])
print('cfg $c', d['ms_per_step'], d['stage_ms']['gn_kernel_ms'])"
done
