run() {
  timeout 900 python bench.py --no-cpu-baseline $2 > gpurun_out/b_ldg.json 2> gpurun_out/b_ldg.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_ldg.json').read().strip().splitlines()[-1])
print('$1', round(d['ms_per_step'],3), round(d['stage_ms']['gn_kernel_ms'],3), round(d['stage_ms']['ll_kernel_ms'],3), round(d['stage_ms']['smooth_ms'],3))" || tail -3 gpurun_out/b_ldg.err
}
run kid_default "--workload kidnap --steps 30 --warmup 25"
SMCL_K2W_CPASYNC=1 run kid_cpasync "--workload kidnap --steps 30 --warmup 25"
run kid_default "--workload kidnap --steps 30 --warmup 25"
run corridor ""
