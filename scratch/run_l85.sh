run() {
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_l.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/b_l.json').read().strip().splitlines()[-1])
print('$1', round(d['ms_per_step'],3), round(d['stage_ms']['ll_kernel_ms'],3))"
}
run default
SMCL_FAST_CFG_LL=L1x85 run L1x85
SMCL_FAST_CFG_LL=L2x84 run L2x84
