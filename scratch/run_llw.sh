run() {
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_ll.json 2> gpurun_out/bench_ll.err
  python -c "
import json
d=json.loads(open('gpurun_out/bench_ll.json').read().strip().splitlines()[-1])
print('$1', d['ms_per_step'], d['stage_ms']['ll_kernel_ms'])" || tail -3 gpurun_out/bench_ll.err
}
run default
for c in 4x16 4x24 4x32; do SMCL_FAST_CFG_LL=$c run w$c; done
