# round 2: K1 with a per-warp candidate queue (records gathered into registers)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for v in "X=1" "SMCL_K1_QUEUE=4x20" "SMCL_K1_QUEUE=2x24" "SMCL_K1_QUEUE=2x28" "SMCL_K1_QUEUE=4x16" "SMCL_K1_QUEUE=4x24"; do
  env $v timeout 600 $B > gpurun_out/r02_k1q.json 2> gpurun_out/r02_k1q.err || tail -5 gpurun_out/r02_k1q.err
  python -c "import json; d=json.load(open('gpurun_out/r02_k1q.json')); print('$v', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items() if k in ('gn_kernel_ms','total_ms')})"
done
SMCL_K1_QUEUE=4x20 timeout 900 python -m pytest tests/test_gpu_likelihood.py tests/test_gpu_parity_step.py -x -q 2>&1 | tail -2
