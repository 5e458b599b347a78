run() {
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_o.json 2> gpurun_out/b_o.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_o.json').read().strip().splitlines()[-1])
print('$1', round(d['ms_per_step'],3), round(d['stage_ms']['svgd_ms'],3), round(d['stage_ms']['ll_kernel_ms'],3))" || tail -3 gpurun_out/b_o.err
}
run base
SMCL_EXP_OVERLAP=1 run overlap
