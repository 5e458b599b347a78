timeout 1500 python -m pytest tests -m gpu -q -k "not outdoor" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>/dev/null
python -c "
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print('default', d['ms_per_step'], d['stage_ms']['gn_kernel_ms'], d['stage_ms']['ll_kernel_ms'])"
for c in 416 L1x84; do
  if [ $c = 416 ]; then unset SMCL_FAST_CFG_LL; else export SMCL_FAST_CFG_LL=$c; fi
  timeout 900 python bench.py --workload kidnap --steps 30 --warmup 25 --no-cpu-baseline > gpurun_out/bench_kid_$c.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_kid_$c.json').read().strip().splitlines()[-1])
print('kid LL $c', d['ms_per_step'], d['stage_ms']['gn_kernel_ms'], d['stage_ms']['ll_kernel_ms'])"
done
