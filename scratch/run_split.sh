run() {
  timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_s.json 2> gpurun_out/b_s.err
  python -c "
import json
d=json.loads(open('gpurun_out/b_s.json').read().strip().splitlines()[-1])
print('$1', round(d['ms_per_step'],3), round(d['stage_ms']['refresh_gather_ms'],3))" || tail -3 gpurun_out/b_s.err
}
run split
SMCL_RG_FUSED=1 run fused
timeout 900 python -m pytest tests -m gpu -q -x -k "neighbor or sharded or stages or golden or filter" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
