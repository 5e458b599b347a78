# round 2: K2 lanes: scan padded in shared memory (no index clamps)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1"; do
  env $v timeout 600 $B > gpurun_out/r02_k2pad.json 2> gpurun_out/r02_k2pad.err || tail -5 gpurun_out/r02_k2pad.err
  python -c "import json; d=json.load(open('gpurun_out/r02_k2pad.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','ll_kernel_ms','total_ms')})"
done
timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py -x -q 2>&1 | tail -2
