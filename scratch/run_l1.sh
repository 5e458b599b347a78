for v in 0 1; do
  if [ $v = 1 ]; then export SMCL_LL_L1=1; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_l1_$v.json 2> /dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_l1_$v.json').read().strip().splitlines()[-1])
print('L1 $v', d['ms_per_step'], d['stage_ms']['ll_kernel_ms'])"
done
