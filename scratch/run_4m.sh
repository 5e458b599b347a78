run() {
  timeout 900 python bench.py --particles 4194304 --scan-points 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4.json 2> gpurun_out/b4.err
  python -c "
import json
d=json.loads(open('gpurun_out/b4.json').read().strip().splitlines()[-1])
print('$1', d['ms_per_step'], {k: round(v,2) for k,v in d['stage_ms'].items()})" || tail -3 gpurun_out/b4.err
}
run default
SMCL_FAST_CFG_LL=416 run ll416
