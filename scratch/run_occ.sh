timeout 1500 python -m pytest tests -m gpu -q -k "not outdoor" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for v in 1 0; do
  if [ $v = 1 ]; then export SMCL_NO_OCC4=1; else unset SMCL_NO_OCC4; fi
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_occ$v.json 2>/dev/null
  python -c "
import json
d=json.loads(open('gpurun_out/bench_occ$v.json').read().strip().splitlines()[-1])
print('no_occ=$v', d['ms_per_step'], d['stage_ms']['ll_kernel_ms'])"
done
