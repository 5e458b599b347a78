# round 2: block-aggregated list/count atomics in the gate split and the solve
timeout 900 python -m pytest tests/test_gpu_stages.py tests/test_gpu_parity_step.py tests/test_gpu_filter.py tests/test_gpu_likelihood.py -x -q -m gpu 2>&1 | tail -3
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "X=1"; do
  env $v timeout 600 $B > gpurun_out/r02_atom.json 2> gpurun_out/r02_atom.err || tail -5 gpurun_out/r02_atom.err
  python -c "import json; d=json.load(open('gpurun_out/r02_atom.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','solve_ms','ll_kernel_ms','total_ms')})"
done
